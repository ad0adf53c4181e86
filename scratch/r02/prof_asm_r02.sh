# ncu metrics of the assembly kernels (plate and C5) after the shared-reciprocal change
cd $GRAFT_REPO_ROOT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread"
python scratch/r02/c5_once.py > gpurun_out/c5_plain.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:"k_bond_rows|k_bond_clamp|k_element_assemble" -s 3 -c 3 --csv --log-file gpurun_out/c5_asm_fp64.csv python scratch/r02/c5_once.py > gpurun_out/ncu_c5.log 2>&1
python scratch/r02/asm_once.py > gpurun_out/asm_plain.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:"k_bond_rows|k_element_assemble" -s 2 -c 2 --csv --log-file gpurun_out/plate_asm_fp64.csv python scratch/r02/asm_once.py > gpurun_out/ncu_plate.log 2>&1
