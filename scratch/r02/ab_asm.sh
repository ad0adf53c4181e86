# A/B of the row-parallel bond pass against the previous tree (scratch/ab_old):
# GPU tests, assembly timing, bit-identity of 4-step (200x120) and 2-step (600K) trajectories
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
for t in new old; do
  d=.; [ $t = old ] && d=scratch/ab_old
  (cd $d && OUT=/tmp/state_$t.npy python $GRAFT_REPO_ROOT/scratch/r02/ab_state.py > $GRAFT_REPO_ROOT/gpurun_out/state_$t.log 2>&1)
  (cd $d && NX=1000 NY=600 K=2 OUT=/tmp/state600_$t.npy python $GRAFT_REPO_ROOT/scratch/r02/ab_state.py > $GRAFT_REPO_ROOT/gpurun_out/state600_$t.log 2>&1)
done
python - <<'PY' > gpurun_out/ab_cmp.txt
import numpy as np
for k in ("state", "state600"):
    a, b = np.load(f"/tmp/{k}_new.npy"), np.load(f"/tmp/{k}_old.npy")
    print(k, "bit-identical" if np.array_equal(a, b) else f"max|diff| {np.abs(a-b).max():.3e}")
PY
