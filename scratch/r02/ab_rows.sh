cd $GRAFT_REPO_ROOT
for v in A0 A1 A1M5; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/rows_$v.so python scratch/r02/asm_micro.py > gpurun_out/rows_$v.json 2>&1; done
