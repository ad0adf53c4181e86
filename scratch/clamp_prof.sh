python scratch/asm_micro.py > gpurun_out/asm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bond_clamp -s 30 -c 1 -o gpurun_out/prof_clamp -f python scratch/asm_micro.py > gpurun_out/ncu_clamp.log 2>&1
python profiles/summarize.py gpurun_out/prof_clamp.ncu-rep > gpurun_out/prof_clamp_summary.txt
