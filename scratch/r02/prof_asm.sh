cd $GRAFT_REPO_ROOT
python scratch/r02/asm_once.py > gpurun_out/asm_once.log 2>&1 && (cd scratch/ab_old && python ../../scratch/r02/asm_once.py >> ../../gpurun_out/asm_once.log 2>&1) &&
ncu --set full --clock-control none --import-source on -k regex:"k_bond_rows|k_bond_assemble|k_element_assemble" -s 2 -c 2 -o gpurun_out/asm_new python scratch/r02/asm_once.py > gpurun_out/ncu_new.log 2>&1
cd scratch/ab_old && ncu --set full --clock-control none --import-source on -k regex:"k_bond_rows|k_bond_assemble|k_element_assemble" -s 2 -c 2 -o ../../gpurun_out/asm_old python ../../scratch/r02/asm_once.py > ../../gpurun_out/ncu_old.log 2>&1
