# problem-sized PCG grids vs the previous library: trajectories bit-identical, mid-size PCG cost
cd $GRAFT_REPO_ROOT
for t in new old; do
  L=""; [ $t = old ] && L="BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/old.so"
  env $L python scratch/r02/rope_pcg.py > gpurun_out/grid_rope_$t.json 2>&1
  env $L K=4 NX=60 NY=36 EPS=1e-6 OUT=/tmp/g_plate_$t.npy python scratch/r02/ab_state.py > gpurun_out/grid_plate_$t.log 2>&1
done
python - <<'PY' > gpurun_out/grid_cmp.txt
import numpy as np
a, b = np.load("/tmp/g_plate_new.npy"), np.load("/tmp/g_plate_old.npy")
print("plate 60x36 4 steps", "bit-identical" if np.array_equal(a, b) else f"max|diff| {np.abs(a-b).max():.3e}")
PY
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
