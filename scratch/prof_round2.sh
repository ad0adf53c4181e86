# in-chain PCG kernels (pcg_micro: 600K plate system, tol 1e-30 so every launch is active)
python scratch/pcg_micro.py > gpurun_out/plain_d.log 2>&1 && \
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_spmv|k_pcg_update|k_pcg_pupdate" -s 60 -c 12 -o gpurun_out/prof_bench_r01d -f python scratch/pcg_micro.py > gpurun_out/ncu_bd.log 2>&1
ncu -i gpurun_out/prof_bench_r01d.ncu-rep --page raw --csv > gpurun_out/prof_bench_r01d_raw.csv
python profiles/summarize.py gpurun_out/prof_bench_r01d.ncu-rep > gpurun_out/prof_bench_r01d_summary.txt
