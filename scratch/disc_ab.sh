for i in 1 2; do python scratch/pcg_micro.py; BDEM_LIB=/root/repo/scratch/lib_disc.so python scratch/pcg_micro.py; done
