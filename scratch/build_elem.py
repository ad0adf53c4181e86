import sys, re
sys.path.insert(0, "/root/repo")
from paper_2308_10459_b200 import _build
src = "/root/repo/paper_2308_10459_b200/csrc/element_kernels.cu"
orig = open(src).read()
try:
    for mb in (1, 2, 3, 4):
        s = orig.replace("__global__ void __launch_bounds__(kThreads) k_element_assemble(",
                         f"__global__ void __launch_bounds__(kThreads, {mb}) k_element_assemble(")
        open(src, "w").write(s)
        print(_build.build(out=f"/root/repo/scratch/lib_elem{mb}.so", force=True, verbose=False))
finally:
    open(src, "w").write(orig)
