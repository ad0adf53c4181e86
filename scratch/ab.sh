for L in scratch/lib_*.so; do BDEM_LIB=$L python scratch/spmv_micro.py 2>&1 | tail -1; done
