"""Builds the in-tree CUDA library `_shardplan_b200.so` for sm_100a.

    python -m paper_2210_02023_b200.build   (or __graft_entry__.build())

Plain nvcc, one object per translation unit (parallel), then one shared
library linked against the static CUDA runtime and NCCL. The .so is written
next to this file so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# SP_BUILD_DIR / SP_LIB_OUT / SP_NVCC_EXTRA: side builds for A/B experiments
BUILD = os.environ.get("SP_BUILD_DIR") or os.path.join(HERE, "_build")
LIB = os.environ.get("SP_LIB_OUT") or os.path.join(HERE, "_shardplan_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# NCCL is not linked: csrc/nccl_loader.h binds it at run time (torch ships
# its own, newer libnccl.so.2 and the two must not collide in one process).
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
              "--expt-relaxed-constexpr", "-Xptxas", "-v,-warn-spills",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _host_compiler_env():
    env = dict(os.environ)
    # The image exports CXX/CC as a wrapper without libgomp; nvcc picks g++
    # from PATH itself, keep PATH's system compiler.
    env.pop("CXX", None)
    env.pop("CC", None)
    return env


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(
            os.path.getmtime(f) for f in [src] + _headers()):
        return obj, ""
    extra = os.environ.get("SP_NVCC_EXTRA", "").split()
    cmd = [nvcc()] + ARCH + NVCC_FLAGS + extra + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True, env=_host_compiler_env())
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + glob.glob(os.path.join(ROOT, "include", "*.h")))


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(_compile, srcs))
    logs = "".join(log for _, log in results)
    if verbose and logs:
        print(logs, file=sys.stderr)
    with open(os.path.join(BUILD, "ptxas.log"), "a") as f:
        f.write(logs)
    objs = [o for o, _ in results]
    if (not os.path.exists(LIB)) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-cudart", "static", "-lrt", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True, env=_host_compiler_env())
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
