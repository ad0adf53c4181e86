cd $GRAFT_REPO_ROOT
for r in 1 2; do for c in 44 58 72; do BDEM_SPMV_CARVEOUT=$c BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/sb.so python scratch/r02/spmv_micro.py > gpurun_out/spmv_sbcv$c\_$r.json 2>&1; done; done
