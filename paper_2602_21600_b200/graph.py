"""Host HNSW graph: builder binding (libaqr_hnsw.so), Alg1 l.17-18 parameter adaptation and a
checksummed graph file.  Not on the timed path: the search consumes the resulting adjacency."""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
import struct
import zlib

import numpy as np

from . import build as _build

_hl = None


def _hlib():
    global _hl
    if _hl is None:
        path = _build.LIB_HNSW
        if not os.path.exists(path):
            raise RuntimeError(f"libaqr_hnsw.so not built ({path})")
        _hl = C.CDLL(path)
        _hl.aqr_hnsw_levels.restype = C.c_int64
        _hl.aqr_hnsw_build.restype = C.c_int
    return _hl


@dataclasses.dataclass
class Graph:
    M: int
    efc: int
    levels: np.ndarray      # int32 [n]
    upper_off: np.ndarray   # int64 [n]
    adj0: np.ndarray        # int32 [n, 2M]
    adj_upper: np.ndarray   # int32 [rows, M]
    entry_point: int
    max_level: int

    @property
    def n(self):
        return self.adj0.shape[0]


def build_hnsw(codes: np.ndarray, M: int, efc: int, level_u: np.ndarray, n_threads: int = 0,
               batch_div: int = 0, flags: int = 0) -> Graph:
    """Deterministic batched HNSW insert over u8 codes [n, d_pad] (Alg1 l.16-22)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n, d_pad = codes.shape
    level_u = np.ascontiguousarray(level_u, dtype=np.float64)
    levels = np.zeros(n, np.int32)
    upper_off = np.zeros(n, np.int64)
    L = _hlib()
    rows = L.aqr_hnsw_levels(level_u.ctypes.data_as(C.c_void_p), C.c_int64(n), C.c_int32(M),
                             levels.ctypes.data_as(C.c_void_p), upper_off.ctypes.data_as(C.c_void_p))
    adj0 = np.empty((n, 2 * M), np.int32)
    adj_upper = np.empty((max(rows, 0), M), np.int32)
    out2 = np.zeros(2, np.int32)
    st = L.aqr_hnsw_build(codes.ctypes.data_as(C.c_void_p), C.c_int64(n), C.c_int32(d_pad),
                          levels.ctypes.data_as(C.c_void_p), upper_off.ctypes.data_as(C.c_void_p), C.c_int32(M),
                          C.c_int32(efc), C.c_int32(n_threads), adj0.ctypes.data_as(C.c_void_p),
                          adj_upper.ctypes.data_as(C.c_void_p) if rows > 0 else None, C.c_int64(rows),
                          out2.ctypes.data_as(C.c_void_p), C.c_int32(batch_div), C.c_int32(flags))
    if st != 0:
        raise RuntimeError(f"aqr_hnsw_build failed ({st})")
    return Graph(M, efc, levels, upper_off, adj0, adj_upper, int(out2[0]), int(out2[1]))


def build_hnsw_gpu(codes, d: int, M: int, efc: int, level_u: np.ndarray, flags: int = 0, batch_div: int = 0,
                   stream=None) -> Graph:
    """aqr_build_graph: the same graph as build_hnsw (byte for byte), built on the GPU (NEXT-1).
    codes: the [n, d_pad] u8 CUDA tensor of aqr_encode; level_u: the seeded uniform draws."""
    from . import lib as _aqr_lib, _dev, _stream, _check
    import torch
    pc = _dev(codes, torch.uint8, "codes")
    n, d_pad = codes.shape
    level_u = np.ascontiguousarray(level_u, dtype=np.float64)
    levels = np.zeros(n, np.int32)
    upper_off = np.zeros(n, np.int64)
    rows = _hlib().aqr_hnsw_levels(level_u.ctypes.data_as(C.c_void_p), C.c_int64(n), C.c_int32(M),
                                   levels.ctypes.data_as(C.c_void_p), upper_off.ctypes.data_as(C.c_void_p))
    adj0 = np.empty((n, 2 * M), np.int32)
    adj_upper = np.empty((max(rows, 0), M), np.int32)
    em = np.zeros(2, np.int32)
    st = _aqr_lib().aqr_build_graph(pc, C.c_int64(n), C.c_int32(d), C.c_int32(d_pad),
                                    levels.ctypes.data_as(C.c_void_p), upper_off.ctypes.data_as(C.c_void_p),
                                    C.c_int64(rows), C.c_int32(M), C.c_int32(efc), C.c_int32(flags),
                                    C.c_int32(batch_div), adj0.ctypes.data_as(C.c_void_p),
                                    adj_upper.ctypes.data_as(C.c_void_p) if rows > 0 else None,
                                    em.ctypes.data_as(C.c_void_p), _stream(stream))
    _check(st, "aqr_build_graph")
    return Graph(M, efc, levels, upper_off, adj0, adj_upper, int(em[0]), int(em[1]))


def density_weights(x_sample: np.ndarray, rho: np.ndarray, literal: bool = False) -> np.ndarray:
    """w_j (Alg1 l.12) -- as printed, w_j = (1/n) sum rho_i is j-independent; R16 takes
    SPEC's density-weighted per-dimension variance, floored at 1e-12, normalised to mean 1.
    literal=True (NEXT-4 variant): the formula as printed, the mean density for every j -- then
    sigma_w = 0, eta = 0, M_i = floor(M0 (1 + delta)) and ef_c = ef_0 (Alg1 l.14, l.17-18)."""
    x = x_sample.astype(np.float64)
    r = rho.astype(np.float64)
    if literal:
        return np.full(x.shape[1], r.mean())
    mu = (r[:, None] * x).sum(0) / r.sum()
    w = (r[:, None] * (x - mu) ** 2).sum(0) / r.sum()
    w = np.maximum(w, 1e-12)
    return w / w.mean()


def eta_of(w: np.ndarray) -> float:
    """eta = sigma_w / w_bar (Alg1 l.14), population std (exactly 0 for constant w)."""
    if np.ptp(w) == 0:
        return 0.0
    return float(np.sqrt(((w - w.mean()) ** 2).mean()) / w.mean())


def adapt_params(M0: int, efc0: int, delta: float, eta: float):
    """M_i = floor(M0 (1 + delta (1 + eta))) (Alg1 l.17);
    ef_c = [efc0 / (1 + delta eta)] read as round-to-nearest, floored at max(16, M_i) (R17)."""
    M = int(math.floor(M0 * (1.0 + delta * (1.0 + eta))))
    efc = int(math.floor(efc0 / (1.0 + delta * eta) + 0.5))
    return M, max(efc, 16, M)


# ------------------------------------------------------------------------------------------
# graph file: magic "AQRG", version, header, arrays, CRC32 ("AQR1" index file)
# ------------------------------------------------------------------------------------------
_MAGIC = b"AQRG"
_VERSION = 1


def save_graph(g: Graph, path: str, tag: str = ""):
    tagb = tag.encode()
    hdr = struct.pack("<4sIqiiiiqI", _MAGIC, _VERSION, g.n, g.M, g.efc, g.entry_point, g.max_level,
                      g.adj_upper.shape[0], len(tagb)) + tagb
    blobs = [hdr, g.levels.astype(np.int32).tobytes(), g.upper_off.astype(np.int64).tobytes(),
             g.adj0.astype(np.int32).tobytes(), g.adj_upper.astype(np.int32).tobytes()]
    crc = 0
    for b in blobs:
        crc = zlib.crc32(b, crc)
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        for b in blobs:
            f.write(b)
        f.write(struct.pack("<I", crc))
    os.replace(tmp, path)


def load_graph(path: str, tag: str | None = None) -> Graph:
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != _MAGIC:
        raise ValueError("not an AQR graph file")
    fixed = struct.calcsize("<4sIqiiiiqI")
    _, ver, n, M, efc, ep, ml, rows, tl = struct.unpack("<4sIqiiiiqI", data[:fixed])
    if ver != _VERSION:
        raise ValueError("graph file version mismatch")
    (crc,) = struct.unpack("<I", data[-4:])
    if zlib.crc32(data[:-4]) != crc:
        raise ValueError("graph file checksum mismatch")
    o = fixed + tl
    ftag = data[fixed:o].decode()
    if tag is not None and ftag != tag:
        raise ValueError("graph file tag mismatch")

    def take(dt, count):
        nonlocal o
        a = np.frombuffer(data, dtype=dt, count=count, offset=o)
        o += a.nbytes
        return a.copy()

    levels = take(np.int32, n)
    upper_off = take(np.int64, n)
    adj0 = take(np.int32, n * 2 * M).reshape(n, 2 * M)
    adj_upper = take(np.int32, rows * M).reshape(rows, M)
    return Graph(M, efc, levels, upper_off, adj0, adj_upper, ep, ml)
