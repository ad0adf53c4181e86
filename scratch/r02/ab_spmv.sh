cd $GRAFT_REPO_ROOT
for v in T0 T1 N1 N1T1; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/spmv_$v.so python scratch/r02/spmv_micro.py > gpurun_out/spmv_$v.json 2>&1; done
(cd scratch/ab_old && python ../../scratch/r02/spmv_micro.py > ../../gpurun_out/spmv_old.json 2>&1)
