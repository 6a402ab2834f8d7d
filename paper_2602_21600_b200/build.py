"""In-tree build of the native libraries (no JIT cache: the .so files travel with the repo).

  libaqr.so       -- the sm_100a CUDA path behind include/aqr.h (nvcc, -gencode
                     arch=compute_100a,code=sm_100a, --fmad=false, -lineinfo, static cudart)
  libaqr_hnsw.so  -- the host HNSW builder (g++, threads)
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_AQR = os.path.join(PKG, "libaqr.so")
LIB_HNSW = os.path.join(PKG, "libaqr_hnsw.so")
CU_SOURCES = ["encode.cu", "search.cu", "merge.cu", "peer.cu", "build.cu", "abi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-Xptxas", "-v"]


def src_hash(deps, flags=()) -> str:
    """16 hex digits of the SHA-256 of the sources (and compiler flags) a library is built from."""
    h = hashlib.sha256()
    for d in deps:
        h.update(os.path.basename(d).encode() + b"\0")
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(" ".join(flags).encode())
    return h.hexdigest()[:16]


def _stamped(target, digest) -> bool:
    """Was `target` built from these sources?  The build embeds "src:<digest>" in the library
    (aqr_version() returns it), so a library pushed or left behind from other sources -- whatever
    its mtime -- is rebuilt."""
    if not os.path.exists(target):
        return False
    with open(target, "rb") as f:
        return f"src:{digest}".encode() in f.read()


def _aqr_deps():
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES]
    return srcs, srcs + [os.path.join(CSRC, "aqr_internal.cuh"), os.path.join(ROOT, "include", "aqr.h")]


def build_aqr(force=False, verbose=False):
    srcs, deps = _aqr_deps()
    digest = src_hash(deps, NVCC_FLAGS)
    if force or not _stamped(LIB_AQR, digest):
        cmd = [NVCC, *NVCC_FLAGS, f"-DAQR_SRC_HASH=\"{digest}\"", "-I", os.path.join(ROOT, "include"), *srcs,
               "-o", LIB_AQR + ".tmp"]
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
    srcs, deps = _aqr_deps()
    flags = [f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")]
    dflags = [f"-D{k}={v}" for k, v in sorted(defines.items())]
    digest = src_hash(deps, flags + dflags)
    if force or not _stamped(out, digest):
        cmd = [NVCC, *flags, *dflags, f"-DAQR_SRC_HASH=\"{digest}\"", "-I", os.path.join(ROOT, "include"),
               *srcs, "-o", out + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed building {out}")
        os.replace(out + ".tmp", out)
    return out


def build_hnsw(force=False):
    src = os.path.join(CSRC, "hnsw_build.cpp")
    flags = ["-O3", "-std=c++17", "-mavx2", "-pthread", "-fPIC", "-shared"]
    digest = src_hash([src], flags)
    if force or not _stamped(LIB_HNSW, digest):
        cmd = ["g++", *flags, f"-DAQR_SRC_HASH=\"{digest}\"", src, "-o", LIB_HNSW + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(LIB_HNSW + ".tmp", LIB_HNSW)
    return LIB_HNSW


def build_all(force=False, verbose=False):
    build_hnsw(force)
    build_aqr(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
