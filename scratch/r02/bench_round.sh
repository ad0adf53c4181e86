# default bench line (driver's parameters), then the launch list of a short run
cd $GRAFT_REPO_ROOT
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo rc=$? >> gpurun_out/bench_r02.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 --no-rot-leg --e2e-steps 0 > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 2500 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 --no-rot-leg --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
