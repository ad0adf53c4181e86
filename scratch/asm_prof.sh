BDEM_LIB=/root/repo/scratch/lib_divnz.so python scratch/asm_micro.py > gpurun_out/asm_plain.log 2>&1 && \
BDEM_LIB=/root/repo/scratch/lib_divnz.so ncu --set full --clock-control none --import-source on -k regex:k_bond_assemble -s 3 -c 1 -o gpurun_out/prof_asm_divnz -f python scratch/asm_micro.py > gpurun_out/ncu_asm.log 2>&1
