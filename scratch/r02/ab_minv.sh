cd $GRAFT_REPO_ROOT
for t in base cert; do BDEM_LIB=$GRAFT_REPO_ROOT/scratch/libs/$t.so OUT=/tmp/m_$t.npz python scratch/r02/minv_cmp.py > gpurun_out/minv_$t.log 2>&1; done
python - <<'PY' > gpurun_out/minv_cmp.txt
import numpy as np
a, b = np.load("/tmp/m_base.npz"), np.load("/tmp/m_cert.npz")
for k in a.files:
    x, y = a[k], b[k]
    same = np.array_equal(x, y)
    print(k, "same" if same else f"DIFF n={int((x != y).sum())} max={np.abs(x - y).max():.3e}")
    if not same and x.ndim == 2:
        cols = np.nonzero((x != y).any(axis=0))[0][:10]
        print("  cols", cols.tolist(), "a", x[:, cols[0]].tolist(), "b", y[:, cols[0]].tolist())
PY
