"""Builds libdct16a.so (the C-ABI library of include/dct16a.h) in-tree with
nvcc for sm_100a.  No torch extension machinery: the library is plain C ABI."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdct16a.so")
BUILD = os.path.join(ROOT, "build", "obj")   # object files (git-ignored), never in csrc/
SOURCES = ["abi.cu", "forward.cu", "codec.cu", "zonal_tpb.cu", "zonal_band.cu", "codec_warp.cu", "codec_uniform.cu", "sweep.cu", "ssim.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "dct16a.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile every source and link libdct16a.so (or `out`, with extra -D
    `defines`, for kernel-variant experiments: e.g. DCT16A_EXPERIMENTS adds the
    round-1 store modes and codec paths).  Objects go to build/obj/ and are
    removed after the link, also when a compile fails."""
    lib = out or LIB
    if out is None and not force and not _stale():
        return LIB
    tag = f".{os.getpid()}.{abs(hash((lib, tuple(defines))))}"
    os.makedirs(BUILD, exist_ok=True)

    def compile_one(s):
        o = os.path.join(BUILD, s.replace(".cu", tag + ".o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, s), "-o", o]
        return s, o, subprocess.run(cmd, capture_output=True, text=True)

    from concurrent.futures import ThreadPoolExecutor
    objs = [os.path.join(BUILD, s.replace(".cu", tag + ".o")) for s in SOURCES]
    try:
        with ThreadPoolExecutor(len(SOURCES)) as ex:
            results = list(ex.map(compile_one, SOURCES))
        for s, o, r in results:
            if verbose or r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode:
                raise RuntimeError(f"nvcc failed on {s}")
        tmp = lib + ".tmp"
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
               "-cudart", "static", "-o", tmp, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, lib)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
