python scratch/asm_micro.py > gpurun_out/asm2_default.json 2>&1
for m in 3; do BDEM_LIB=/root/repo/scratch/lib_asm2_m$m.so python scratch/asm_micro.py > gpurun_out/asm2_m$m.json 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests2.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests2.log
