for i in 1 2; do for it in 1 2 6 12; do BDEM_LIB=/root/repo/scratch/lib_pu$it.so python scratch/pcg_micro.py; done; done
