for L in prev reorder reorder_m3 prev; do BDEM_LIB=/root/repo/scratch/lib_$L.so python scratch/asm_micro.py > gpurun_out/asm3_$L.json 2>&1; done
