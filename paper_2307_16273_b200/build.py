"""Build libzkdl.so in-tree for sm_100a (nvcc, one object per translation unit, in parallel).

    python -m paper_2307_16273_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OBJ = os.path.join(os.path.dirname(HERE), "build", "obj")
SO = os.path.join(HERE, "libzkdl.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "177"]
# ZKDL_FR64=0 builds the hot product bodies with the integer CIOS instead of the FP64-pipe product (A/B)
if os.environ.get("ZKDL_FR64") is not None:
    FLAGS += [f"-DZKDL_FR64={int(os.environ['ZKDL_FR64'])}"]
# ZKDL_DEFS="NAME=VALUE ...": extra compile-time settings for A/B builds (e.g. ZKDL_IR_LB_T, ZKDL_IR_LB_B)
FLAGS += [f"-D{d}" for d in os.environ.get("ZKDL_DEFS", "").split() if d]


def _deps():
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return max((os.path.getmtime(h) for h in hdrs), default=0.0)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _deps()):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-I", INCLUDE, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    newest_src = max([os.path.getmtime(s) for s in srcs] + [_deps()])
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= newest_src:
        return SO
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", SO, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print("built", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv)
