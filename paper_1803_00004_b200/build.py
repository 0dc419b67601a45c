"""Builds libbf.so in-tree with nvcc for sm_100a (the product library; no torch linkage).

    python -m paper_1803_00004_b200.build [--force] [-v]     # or via __graft_entry__.build()

Each translation unit compiles to an object file in parallel (the kernel TUs hold many template
instantiations), then nvcc links the shared library.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libbf.so")
SOURCES = ["bf_plan.cpp", "bf_apply.cu", "bf_k_band.cu", "bf_k_ws.cu", "bf_k_ws2.cu", "bf_k_ws2m_u8.cu",
           "bf_k_ws2m_f32.cu", "bf_k_ws2c.cu", "bf_k_lit.cu", "bf_k_cache.cu",
           "bf_k_repair.cu"]
HEADERS = ["bf_internal.h", "bf_params.h", "bf_device.cuh", "bf_walk.cuh", "bf_ws2.cuh", "bf_tm.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps_mtime() -> float:
    paths = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(HERE, "..", "include", "bf.h")]
    return max(os.path.getmtime(p) for p in paths)


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return _deps_mtime() > t or any(os.path.getmtime(os.path.join(CSRC, s)) > t for s in SOURCES)


def _compile(src: str, force: bool, ptxas_v: bool) -> tuple:
    obj = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
    s = os.path.join(CSRC, src)
    if (not force and os.path.exists(obj) and os.path.getmtime(obj) >= os.path.getmtime(s)
            and os.path.getmtime(obj) >= _deps_mtime()):
        return obj, ""
    cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", obj + ".tmp", s]
    if ptxas_v and src.endswith(".cu"):
        cmd[1:1] = ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        res = list(ex.map(lambda s: _compile(s, force, ptxas_v), SOURCES))
    if verbose or ptxas_v:
        for _, err in res:
            sys.stdout.write(err)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *[o for o, _ in res],
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv)
    print(LIB)
