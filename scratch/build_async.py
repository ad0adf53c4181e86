import sys
sys.path.insert(0, "/root/repo")
from paper_2308_10459_b200 import _build
variants = {"base": [], "a4s12": ["-DBDEM_SPMV_ASYNC=1", "-DBDEM_ASYNC_WARPS=4", "-DBDEM_ASYNC_SLOTS=12"],
            "a6s12": ["-DBDEM_SPMV_ASYNC=1", "-DBDEM_ASYNC_WARPS=6", "-DBDEM_ASYNC_SLOTS=12"],
            "a4s8": ["-DBDEM_SPMV_ASYNC=1", "-DBDEM_ASYNC_WARPS=4", "-DBDEM_ASYNC_SLOTS=8"],
            "a8s16": ["-DBDEM_SPMV_ASYNC=1", "-DBDEM_ASYNC_WARPS=8", "-DBDEM_ASYNC_SLOTS=16"],
            "a12s12": ["-DBDEM_SPMV_ASYNC=1", "-DBDEM_ASYNC_WARPS=12", "-DBDEM_ASYNC_SLOTS=12"]}
for name, flags in variants.items():
    try:
        print(_build.build(extra=flags, out=f"/root/repo/scratch/lib_{name}.so"))
    except Exception as e:
        print("FAIL", name, str(e)[-500:])
