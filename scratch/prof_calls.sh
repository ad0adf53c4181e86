# which kernels of the Newton loop still execute FP64-division slow-path calls
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-c5 --no-rot-leg"
$CMD > gpurun_out/plain_calls.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_element_assemble|k_bond_energy|k_element_energy|k_bond_assemble|k_direction|k_pair" -s 10 -c 8 -o gpurun_out/prof_calls -f $CMD > gpurun_out/ncu_calls.log 2>&1
python profiles/summarize.py gpurun_out/prof_calls.ncu-rep > gpurun_out/prof_calls_summary.txt
