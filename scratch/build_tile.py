"""Build tiled-SpMV variants into scratch/lib_tile_*.so for A/B on the GPU."""
import os, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.getcwd())
from paper_2308_10459_b200 import _build
# name: (TS, NW, STAGES, MINB, DIAG)
V = {"t1w8s3m2d1": (1, 8, 3, 2, 1), "t1w8s2m3d1": (1, 8, 2, 3, 1), "t1w4s3m2d1": (1, 4, 3, 2, 1),
     "t1w4s2m3d0": (1, 4, 2, 3, 0), "t2w8s3m1d1": (2, 8, 3, 1, 1), "t2w16s3m1d1": (2, 16, 3, 1, 1),
     "t4w16s2m1d0": (4, 16, 2, 1, 0), "t1w8s4m1d1": (1, 8, 4, 1, 1)}
if len(sys.argv) > 1:
    V = {k: v for k, v in V.items() if k in sys.argv[1:]}
def one(kv):
    k, (ts, nw, st, mb, dg) = kv
    out = os.path.join("scratch", f"lib_tile_{k}.so")
    _build.build(extra=[f"-DBDEM_TILE_TS={ts}", f"-DBDEM_TILE_NW={nw}", f"-DBDEM_TILE_STAGES={st}",
                        f"-DBDEM_TILE_MINB={mb}", f"-DBDEM_TILE_DIAG={dg}"], out=out)
    return out
with ThreadPoolExecutor(6) as ex:
    for o in ex.map(one, V.items()):
        print(o)
