# assembly timing of several library builds: scratch/libs/<name>.so for each argument
# ("base" = the in-tree library)
cd $GRAFT_REPO_ROOT
for t in "$@"; do
  L="BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/$t.so"; [ $t = base ] && L="BDEM_X=0"
  env $L python scratch/r02/asm_micro.py > gpurun_out/asm_$t.json 2> gpurun_out/asm_$t.err
  echo $t; tail -1 gpurun_out/asm_$t.json
done
