cd $GRAFT_REPO_ROOT
python scratch/r02/asm_micro.py > gpurun_out/rows_base.json 2>&1
for v in M6 M5 M4; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/rows_$v.so python scratch/r02/asm_micro.py > gpurun_out/rows_$v.json 2>&1; done
cd scratch/ab_old
python ../../scratch/r02/asm_micro.py > ../../gpurun_out/rows_old.json 2>&1
for v in M6 M5 M4; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/old_$v.so python ../../scratch/r02/asm_micro.py > ../../gpurun_out/rows_old$v.json 2>&1; done
