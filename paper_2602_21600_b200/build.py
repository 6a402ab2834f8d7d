"""In-tree build of the native libraries (no JIT cache: the .so files travel with the repo).

  libaqr.so       -- the sm_100a CUDA path behind include/aqr.h (nvcc, -gencode
                     arch=compute_100a,code=sm_100a, --fmad=false, -lineinfo, static cudart)
  libaqr_hnsw.so  -- the host HNSW builder (g++, threads)
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_AQR = os.path.join(PKG, "libaqr.so")
LIB_HNSW = os.path.join(PKG, "libaqr_hnsw.so")
CU_SOURCES = ["encode.cu", "search.cu", "merge.cu", "abi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-Xptxas", "-v"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_aqr(force=False, verbose=False):
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES]
    deps = srcs + [os.path.join(CSRC, "aqr_internal.cuh"), os.path.join(ROOT, "include", "aqr.h")]
    if force or _stale(LIB_AQR, deps):
        cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), *srcs, "-o", LIB_AQR + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libaqr.so")
        with open(os.path.join(PKG, "ptxas.log"), "w") as f:
            f.write(r.stderr)
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(LIB_AQR + ".tmp", LIB_AQR)
    return LIB_AQR


def build_variant(name: str, defines: dict, force=False):
    """Build libaqr_<name>.so with -D overrides of the compile-time tuning knobs (tools/perf.py)."""
    out = os.path.join(PKG, f"libaqr_{name}.so")
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES]
    deps = srcs + [os.path.join(CSRC, "aqr_internal.cuh"), os.path.join(ROOT, "include", "aqr.h")]
    if force or _stale(out, deps):
        flags = [f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")]
        cmd = [NVCC, *flags, *[f"-D{k}={v}" for k, v in defines.items()], "-I", os.path.join(ROOT, "include"),
               *srcs, "-o", out + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed building {out}")
        os.replace(out + ".tmp", out)
    return out


def build_hnsw(force=False):
    src = os.path.join(CSRC, "hnsw_build.cpp")
    if force or _stale(LIB_HNSW, [src]):
        cmd = ["g++", "-O3", "-std=c++17", "-mavx2", "-pthread", "-fPIC", "-shared", src, "-o", LIB_HNSW + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(LIB_HNSW + ".tmp", LIB_HNSW)
    return LIB_HNSW


def build_all(force=False, verbose=False):
    build_hnsw(force)
    build_aqr(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
