import sys, re
sys.path.insert(0, "/root/repo")
from paper_2308_10459_b200 import _build
src = "/root/repo/paper_2308_10459_b200/csrc/bond_kernels.cu"
orig = open(src).read()
try:
    for mb in (3, 4, 5, 6):
        s = re.sub(r"__launch_bounds__\(128(, \d+)?\) k_bond_assemble\(", f"__launch_bounds__(128, {mb}) k_bond_assemble(", orig)
        open(src, "w").write(s)
        print(_build.build(out=f"/root/repo/scratch/lib_asmb{mb}.so", force=True))
finally:
    open(src, "w").write(orig)
