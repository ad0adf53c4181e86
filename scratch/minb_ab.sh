python scratch/pcg_micro.py
for m in 6 7; do BDEM_LIB=/root/repo/scratch/lib_m$m.so python scratch/pcg_micro.py; done
