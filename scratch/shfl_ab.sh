for L in /root/repo/scratch/lib_shfl_m6.so /root/repo/scratch/lib_shfl_m8.so; do for ro in id strip; do BDEM_LIB=$L BDEM_ROW_ORDER=$ro python scratch/shfl_micro.py; done; done
