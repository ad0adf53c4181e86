# shared-reciprocal quotients vs IEEE division (scratch/libs/ieee.so = HEAD):
# trajectories, GPU tests, assembly timing
cd $GRAFT_REPO_ROOT
for t in new ieee; do
  L=""; [ $t = ieee ] && L="BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/ieee.so"
  env $L OUT=/tmp/s_$t.npy python scratch/r02/ab_state.py > gpurun_out/div_state_$t.log 2>&1
  env $L NX=1000 NY=600 K=2 OUT=/tmp/s600_$t.npy python scratch/r02/ab_state.py > gpurun_out/div_state600_$t.log 2>&1
  env $L python scratch/r02/asm_micro.py > gpurun_out/div_asm_$t.json 2>&1
done
python - <<'PY' > gpurun_out/div_cmp.txt
import numpy as np
for k in ("s", "s600"):
    a, b = np.load(f"/tmp/{k}_new.npy"), np.load(f"/tmp/{k}_ieee.npy")
    print(k, "bit-identical" if np.array_equal(a, b) else f"max|diff| {np.abs(a-b).max():.3e} rel {np.abs(a-b).max()/np.abs(b).max():.3e}")
PY
python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
