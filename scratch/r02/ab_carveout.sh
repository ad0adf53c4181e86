# SpMV timing against the shared-memory carveout preference of k_spmv
cd $GRAFT_REPO_ROOT
for r in 1 2; do
BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/base.so python scratch/r02/spmv_micro.py > gpurun_out/spmv_base_$r.json 2>&1
for c in 100 60 50 25; do BDEM_SPMV_CARVEOUT=$c BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/cv.so python scratch/r02/spmv_micro.py > gpurun_out/spmv_cv$c\_$r.json 2>&1; done; done
