"""Build libmgnn.so (sm_100a) in-tree with nvcc.

`python -m paper_2410_22697_b200.build` or `build()` from __graft_entry__.
Each .cu unit is compiled to an object with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
(no --use_fast_math: fp32 scores must stay IEEE RN with denormals, DESIGN R#12)
and linked into a shared library next to this file.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmgnn.so")
LIB_CHECKED = os.path.join(HERE, "libmgnn_checked.so")
UNITS = ["api.cu", "api_sage.cu", "partition.cu", "sample.cu", "gather.cu", "score.cu", "sort.cu", "load.cu", "sage.cu", "train.cu"]
HEADERS = ["common.cuh", "launch.h", "umma.cuh", "ctx.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("MGNN_NVCC_EXTRA", "").split()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-fmad=false", "-ftz=false",
         "-prec-div=true", "-prec-sqrt=true", f"-I{os.path.join(ROOT, 'include')}"] + EXTRA


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """checked=True builds libmgnn_checked.so with the device bounds checks (-DMGNN_CHECKS: every
    MGNN_CHECK traps with a message) -- the debug library the test suite can load through MGNN_LIB."""
    objdir = os.path.join(HERE, "build_checked" if checked else "build")
    os.makedirs(objdir, exist_ok=True)
    lib = LIB_CHECKED if checked else LIB
    flags = FLAGS + (["-DMGNN_CHECKS"] if checked else [])
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "mgnn.h")]
    jobs = []
    for u in UNITS:
        src = os.path.join(CSRC, u)
        obj = os.path.join(objdir, u.replace(".cu", ".o"))
        if force or _stale(obj, [src] + hdrs):
            jobs.append([NVCC, *flags, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)

    with ThreadPoolExecutor(max_workers=min(6, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(objdir, u.replace(".cu", ".o")) for u in UNITS]
    if force or jobs or _stale(lib, objs):
        tmp = lib + f".tmp{os.getpid()}"
        run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp, "-lcudart"])
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
