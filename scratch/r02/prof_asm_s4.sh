cd $GRAFT_REPO_ROOT
python scratch/r02/asm_once.py > gpurun_out/asm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bond_rows|k_element_assemble" -s 2 -c 2 -o gpurun_out/asm_s4 -f python scratch/r02/asm_once.py > gpurun_out/ncu_asm.log 2>&1
tail -2 gpurun_out/ncu_asm.log
