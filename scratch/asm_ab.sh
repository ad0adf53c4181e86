for L in "$@"; do BDEM_LIB=$L python scratch/asm_micro.py; done
