# FP64 DFMA peak, eigen-clamp FP64 counters (every rotation block of the
# plate perturbed, all 3.59M blocks through k_bond_clamp), and the mutation
# check of the rotation parity tests (retraction step scaled by 1 + 1e-9)
set -x
mkdir -p gpurun_out/r02n
./scratch/r02/fp64/fp64_peak > gpurun_out/r02n/fp64_peak.json
timeout 900 python -m pytest tests/test_gpu_parity.py -k "trajectory" -q -p no:cacheprovider > gpurun_out/r02n/traj_tests.log 2>&1; echo rc=$? >> gpurun_out/r02n/traj_tests.log
BDEM_LIB=$PWD/scratch/libs/mut_retract.so timeout 900 python -m pytest tests/test_gpu_parity.py -k "trajectory and rope" -q -p no:cacheprovider > gpurun_out/r02n/mutation_rope.log 2>&1; echo rc=$? >> gpurun_out/r02n/mutation_rope.log
python scratch/r02/asm_micro.py > gpurun_out/r02n/asm_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bond_clamp|k_bond_assemble" -s 94 -c 4 --csv --log-file gpurun_out/r02n/clamp_fp64.csv python scratch/r02/asm_micro.py > gpurun_out/r02n/ncu.log 2>&1
echo done
