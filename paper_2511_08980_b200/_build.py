"""Build libfdsdf.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build() and the tests."""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libfdsdf.so")
BUILD = os.path.join(ROOT, "build")
SOURCES = ["api.cu", "fwd.cu", "bwd.cu", "wgrad.cu", "tcprobe.cu", "fwd_tc.cu", "bwd_tc.cu", "wgrad_tc.cu", "train.cu", "bwdl_tc.cu", "mesh.cu"]
HEADERS = ["common.cuh", "act.cuh", "tile.cuh", "kernels.cuh", "tc.cuh", "fdepi.cuh", "tcmlp.cuh", "tcpair.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("FDSDF_NVCC_EXTRA", "").split()  # debug builds only (e.g. -DFDSDF_PHASE_TIMING)
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-diag-suppress", "177"]


def _newest_input():
    paths = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    paths.append(os.path.join(ROOT, "include", "fdsdf.h"))
    paths.append(os.path.abspath(__file__))
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False, lib: str = LIB, build_dir: str = BUILD) -> str:
    """Compile every .cu for sm_100a and link libfdsdf.so; returns its path.  `lib` / `build_dir`
    redirect the output (compile-time variants for A/B timing, see scripts/build_variant.py)."""
    LIB, BUILD = lib, build_dir
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_input():
        return LIB
    os.makedirs(BUILD, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *EXTRA, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(BUILD, src.replace(".cu", ".ptxas.log"))
        with open(log, "w") as fh:
            fh.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, LIB)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
