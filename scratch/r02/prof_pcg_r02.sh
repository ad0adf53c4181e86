# ncu --set full of the in-chain PCG kernels (600K plate system), current library
cd $GRAFT_REPO_ROOT
python scratch/pcg_micro.py > gpurun_out/pcg_plain.log 2>&1 && \
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_spmv|k_pcg_update|k_pcg_pupdate" -s 60 -c 12 -o gpurun_out/prof_pcg_r02 -f python scratch/pcg_micro.py > gpurun_out/ncu_pcg.log 2>&1
