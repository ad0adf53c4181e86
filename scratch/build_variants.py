import sys, os
sys.path.insert(0, "/root/repo")
from paper_2308_10459_b200 import _build
for spec in sys.argv[1:]:
    w, b, m = spec.split(",")
    out = f"/root/repo/scratch/lib_w{w}_b{b}_m{m}.so"
    try:
        _build.build(extra=[f"-DBDEM_SPMV_WARPS={w}", f"-DBDEM_SPMV_BLOCKED={b}", f"-DBDEM_SPMV_MINB={m}"], out=out)
        print("ok", out)
    except Exception as ex:
        print("FAIL", out, str(ex)[-300:])
