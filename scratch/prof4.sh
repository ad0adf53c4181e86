CMD="python scratch/spmv_micro.py"
$CMD > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_spmv|k_pcg_update|k_pcg_pupdate|k_bond_assemble|k_element_assemble|k_bond_energy" -s 10 -c 6 -o gpurun_out/prof_r01_v5 $CMD > gpurun_out/ncu5.log 2>&1; tail -2 gpurun_out/ncu5.log
