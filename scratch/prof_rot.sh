CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-c5 --no-rot-leg"
BDEM_ROT_SKIP=1 $CMD > gpurun_out/plain_rot.log 2>&1 && \
BDEM_ROT_SKIP=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -s 2000 -c 900 --csv --log-file gpurun_out/launches_rot.csv $CMD > gpurun_out/ncu_rot.log 2>&1
python profiles/launch_shares.py gpurun_out/launches_rot.csv > gpurun_out/launches_rot_shares.txt
