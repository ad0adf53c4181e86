# A/B of two library builds (scratch/libs/base.so vs scratch/libs/$1.so):
# assembly timing + checksums, 200x120 and 600K trajectories
cd $GRAFT_REPO_ROOT
V=${1:-cert}
for t in base $V; do
  L="BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/$t.so"
  env $L python scratch/r02/asm_micro.py > gpurun_out/ab_asm_$t.json 2>&1
  env $L OUT=/tmp/s_$t.npy python scratch/r02/ab_state.py > gpurun_out/ab_state_$t.log 2>&1
  env $L NX=1000 NY=600 K=2 OUT=/tmp/s600_$t.npy python scratch/r02/ab_state.py > gpurun_out/ab_state600_$t.log 2>&1
done
V=$V python - <<'PY' > gpurun_out/ab_cmp.txt
import numpy as np, os
v = os.environ["V"]
for k in ("s", "s600"):
    a, b = np.load(f"/tmp/{k}_{v}.npy"), np.load(f"/tmp/{k}_base.npy")
    print(k, "bit-identical" if np.array_equal(a, b) else f"max|diff| {np.abs(a-b).max():.3e}")
PY
