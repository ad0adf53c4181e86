for i in 1 2; do python scratch/pcg_micro.py; BDEM_LIB=/root/repo/scratch/lib_stream.so python scratch/pcg_micro.py; BDEM_LIB=/root/repo/scratch/lib_stream2.so python scratch/pcg_micro.py; done
