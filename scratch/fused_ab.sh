for i in 1 2; do python scratch/pcg_micro.py; BDEM_FUSED_UPD=1 python scratch/pcg_micro.py; done
