for L in /root/repo/scratch/lib_prev.so /root/repo/scratch/lib_unroll2.so; do
BDEM_LIB=$L python scratch/pcg_micro.py
BDEM_LIB=$L BDEM_ROT_SKIP=1 python scratch/pcg_micro.py
done
