"""Build the sm_100a CUDA library in-tree (``lib/libbdem_sm100.so``).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the build
container; the resulting ``.so`` travels to the GPU box with the repo.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
OBJDIR = os.path.join(LIBDIR, "obj")
LIBNAME = "libbdem_sm100.so"
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-Xptxas", "-warn-spills"]


def _nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def lib_path() -> str:
    # BDEM_LIB selects an alternative build of the same library (A/B tests)
    return os.environ.get("BDEM_LIB") or os.path.join(LIBDIR, LIBNAME)


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, extra=None, out=None) -> str:
    """Compile csrc/*.cu for sm_100a and link lib/libbdem_sm100.so.

    ``extra`` adds nvcc flags and ``out`` redirects the library (A/B builds
    of kernel variants, selected at run time with BDEM_LIB)."""
    objdir = OBJDIR if out is None else out + ".obj"
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(INCLUDE, "bdem_sm100.h")]
    objs, jobs = [], []
    for src in sources:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [nvcc, *ARCH, *FLAGS, *(extra or []), "-I", INCLUDE, "-c", src, "-o", obj]
            if verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stdout + r.stderr

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for log in ex.map(run, jobs):
            if verbose and log:
                print(log)
    target = out or os.path.join(LIBDIR, LIBNAME)
    if force or jobs or _stale(target, objs):
        run([nvcc, *ARCH, "-shared", "-o", target, *objs])
    return target


if __name__ == "__main__":
    import sys
    extra = [a for a in sys.argv[1:] if a.startswith("-D")]
    out = next((a[6:] for a in sys.argv[1:] if a.startswith("--out=")), None)
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, extra=extra, out=out))
