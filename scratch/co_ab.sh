python scratch/pcg_micro.py
for c in 0 25 50 100; do BDEM_LIB=/root/repo/scratch/lib_co$c.so python scratch/pcg_micro.py; done
python scratch/spmv_micro.py
for c in 0 25 50 100; do BDEM_LIB=/root/repo/scratch/lib_co$c.so python scratch/spmv_micro.py; done
