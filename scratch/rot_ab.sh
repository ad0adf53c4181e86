timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rot_skip or fused or newton_solve" > gpurun_out/rot_tests.log 2>&1; echo rc=$? >> gpurun_out/rot_tests.log
python scratch/pcg_micro.py > gpurun_out/rot_pcg.out 2>&1
BDEM_ROT_SKIP=1 python scratch/pcg_micro.py >> gpurun_out/rot_pcg.out 2>&1
