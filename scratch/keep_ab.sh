for i in 1 2; do BDEM_LIB=/root/repo/scratch/lib_keep.so python scratch/pcg_micro.py; BDEM_LIB=/root/repo/scratch/lib_keep2.so python scratch/pcg_micro.py; done
