# A/B of several SpMV library builds: scratch/libs/{base,$@}.so, 2 rounds each
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in base "$@"; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/$v.so python scratch/r02/spmv_micro.py > gpurun_out/spmv_${v}_$r.json 2>&1; done; done
