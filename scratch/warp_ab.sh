for i in 1 2; do python scratch/pcg_micro.py; BDEM_SPMV_TILE=5 python scratch/pcg_micro.py; done
python scratch/spmv_micro.py; BDEM_SPMV_TILE=5 python scratch/spmv_micro.py
