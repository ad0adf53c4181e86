cd $GRAFT_REPO_ROOT
V=${1:-cert3}
for t in base $V; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/$t.so OUT=/tmp/m_$t.npz python scratch/r02/minv_cmp.py > gpurun_out/minv_$t.log 2>&1; done
V=$V python - <<'PY' > gpurun_out/minv_cmp.txt
import numpy as np, os
a, b = np.load("/tmp/m_base.npz"), np.load(f"/tmp/m_{os.environ['V']}.npz")
for k in a.files:
    x, y = a[k], b[k]
    print(k, "same" if np.array_equal(x, y) else f"DIFF n={int((x != y).sum())} max={np.abs(x - y).max():.3e}")
PY
bash scratch/r02/ab_lib.sh $V
