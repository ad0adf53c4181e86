cd $GRAFT_REPO_ROOT
V=${1:-hdr}
for r in 1 2; do for v in base $V; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/$v.so python scratch/r02/spmv_micro.py > gpurun_out/spmv_${v}_$r.json 2>&1; done; done
