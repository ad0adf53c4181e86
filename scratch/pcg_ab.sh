python scratch/pcg_micro.py
BDEM_FUSED_UPD=0 python scratch/pcg_micro.py
BDEM_PDL=0 python scratch/pcg_micro.py
BDEM_PDL=0 BDEM_FUSED_UPD=0 python scratch/pcg_micro.py
