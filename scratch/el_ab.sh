for i in 1 2; do BDEM_LIB=/root/repo/scratch/lib_prev.so python scratch/spmv_micro.py; BDEM_LIB=/root/repo/scratch/lib_new.so python scratch/spmv_micro.py; done
