cd $GRAFT_REPO_ROOT
python scratch/r02/spmv_micro.py > gpurun_out/spmv_base.json 2>&1
for v in B7 B6 T7 NT7 NT6 N7; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/spmv_$v.so python scratch/r02/spmv_micro.py > gpurun_out/spmv_$v.json 2>&1; done
python scratch/r02/asm_micro.py > gpurun_out/el_base.json 2>&1
BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/el_J1.so python scratch/r02/asm_micro.py > gpurun_out/el_J1.json 2>&1
bash scratch/r02/prof_r02.sh
