"""Build SpMV variants into scratch/lib_*.so for A/B on the GPU."""
import os, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.getcwd())
from paper_2308_10459_b200 import _build
# name: extra flags
V = {"blocked": ["-DBDEM_SPMV_BLOCKED=1"],
     "wave_m6": ["-DBDEM_WAVE_MINB=6"], "wave_m5": ["-DBDEM_WAVE_MINB=5"],
     "sym_t2w8m3": ["-DBDEM_SYM_TS=2", "-DBDEM_SYM_NW=8", "-DBDEM_SYM_MINB=3"],
     "sym_t2w4m6": ["-DBDEM_SYM_TS=2", "-DBDEM_SYM_NW=4", "-DBDEM_SYM_MINB=6"],
     "sym_t4w16m1": ["-DBDEM_SYM_TS=4", "-DBDEM_SYM_NW=16", "-DBDEM_SYM_MINB=1"],
     "sym_t4w8m3": ["-DBDEM_SYM_TS=4", "-DBDEM_SYM_NW=8", "-DBDEM_SYM_MINB=3"],
     "t4w16s2m1": ["-DBDEM_TILE_TS=4", "-DBDEM_TILE_NW=16", "-DBDEM_TILE_STAGES=2", "-DBDEM_TILE_MINB=1", "-DBDEM_TILE_DIAG=0"],
     "t2w8s2m2": ["-DBDEM_TILE_TS=2", "-DBDEM_TILE_NW=8", "-DBDEM_TILE_STAGES=2", "-DBDEM_TILE_MINB=2", "-DBDEM_TILE_DIAG=0"],
     "t2w8s3m1": ["-DBDEM_TILE_TS=2", "-DBDEM_TILE_NW=8", "-DBDEM_TILE_STAGES=3", "-DBDEM_TILE_MINB=1", "-DBDEM_TILE_DIAG=1"],
     "t4w8s2m1": ["-DBDEM_TILE_TS=4", "-DBDEM_TILE_NW=8", "-DBDEM_TILE_STAGES=2", "-DBDEM_TILE_MINB=1", "-DBDEM_TILE_DIAG=0"]}
if len(sys.argv) > 1:
    V = {k: v for k, v in V.items() if k in sys.argv[1:]}
def one(kv):
    k, flags = kv
    out = os.path.join("scratch", f"lib_{k}.so")
    _build.build(extra=flags, out=out)
    return out
with ThreadPoolExecutor(5) as ex:
    for o in ex.map(one, V.items()):
        print(o)
