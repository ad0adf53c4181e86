cd $GRAFT_REPO_ROOT
python scratch/r02/spmv_micro.py > gpurun_out/spmv_base.json 2>&1
for v in PIN100 PIN150 PIN200 PIN250; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/spmv_$v.so python scratch/r02/spmv_micro.py > gpurun_out/spmv_$v.json 2>&1; done
python scratch/r02/spmv_micro.py > gpurun_out/spmv_base2.json 2>&1
