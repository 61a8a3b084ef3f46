"""In-tree build of libsketchcu.so (sm_100a) with nvcc.

The .so lands in paper_1511_00152_b200/_lib/. It is git-ignored but travels to the
GPU box with the gpurun snapshot. Objects are rebuilt only when a source or header
is newer than the object.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_lib")
SO = os.path.join(OUT, "libsketchcu.so")
SOURCES = ["capi.cu", "sketch.cu", "moments.cu", "cov_tc.cu", "kmeans.cu", "kmeans_tc.cu", "formats.cu", "dense.cu", "gather.cu", "lloyd.cu", "comm.cu", "eig.cu"]
HEADERS = [os.path.join(CSRC, "common.cuh"), os.path.join(ROOT, "include", "sketchcu.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include")]
# experiments only: extra nvcc flags, e.g. SKC_EXTRA_NVCC_FLAGS="-DSKC_GATHER_STAGES=3"
FLAGS += os.environ.get("SKC_EXTRA_NVCC_FLAGS", "").split()


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str) -> str:
    obj = os.path.join(OUT, os.path.splitext(src)[0] + ".o")
    path = os.path.join(CSRC, src)
    if _newer(obj, [path] + HEADERS):
        cmd = [NVCC, *ARCH, *FLAGS, "-c", path, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(os.path.join(OUT, os.path.splitext(src)[0] + ".ptxas.log"), "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if _newer(SO, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", SO, *objs, "-lcudart", "-ldl", "-lcusolver"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    if verbose:
        print(SO)
    return SO


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
