python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -3
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain3.log 2>&1 && tail -c 1600 gpurun_out/plain3.log && \
ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 200 -c 1 -o gpurun_out/prof_spmv3 $CMD > gpurun_out/ncu_s3.log 2>&1; tail -2 gpurun_out/ncu_s3.log
