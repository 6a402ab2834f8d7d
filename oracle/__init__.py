"""CPU oracle for the AQR-HNSW hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  It shares no code with paper_2602_21600_b200 (the product) and
imports nothing from it.  The arithmetic lives in aqr_oracle.c (plain C, single thread,
-O2 -ffp-contract=off); this module only marshals numpy arrays through ctypes.

Paper citations are in aqr_oracle.c next to each function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "aqr_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
NCOUNT = 10
COUNTER_NAMES = ["expansions", "deg_sum", "evals", "upper_exp", "upper_deg_sum", "upper_evals",
                 "n_coarse", "depth", "early_term", "n_asym"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               _SRC, "-o", _SO + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.or_delta.restype = C.c_double
        _lib.or_percentile_sorted.restype = C.c_double
        _lib.or_build_upper_rows.restype = C.c_int64
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class _Index(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("d_pad", C.c_int32), ("metric", C.c_int32),
                ("codes", C.c_void_p), ("base", C.c_void_p), ("min_f", C.c_void_p),
                ("scale_f", C.c_void_p), ("max_level", C.c_int32), ("entry_point", C.c_int32),
                ("cap0", C.c_int32), ("adj0", C.c_void_p), ("capu", C.c_int32),
                ("upper_off", C.c_void_p), ("adj_upper", C.c_void_p), ("levels", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("k", C.c_int32), ("ef", C.c_int32), ("n_coarse", C.c_int32), ("n_rerank", C.c_int32),
                ("tau_gap", C.c_double), ("tau_ratio", C.c_double), ("early_term", C.c_int32),
                ("assemble_mode", C.c_int32), ("beam_form", C.c_int32), ("traversal", C.c_int32),
                ("tau_spread", C.c_double)]


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ------------------------------------------------------------------------------------------
# build phase
# ------------------------------------------------------------------------------------------

def density(x, sample, k=10, eps=1e-6):
    x = _c(x, np.float32)
    sample = _c(sample, np.int32)
    rho = np.zeros(len(sample), np.float64)
    st = lib().or_density(_p(x), C.c_int64(x.shape[0]), C.c_int32(x.shape[1]), _p(sample),
                          C.c_int32(len(sample)), C.c_int32(k), C.c_double(eps), _p(rho))
    if st:
        raise ValueError(f"or_density status {st}")
    return rho


def delta(rho, eps=1e-6):
    rho = _c(rho, np.float64)
    return lib().or_delta(_p(rho), C.c_int32(len(rho)), C.c_double(eps))


def percentile_sorted(s, P):
    s = _c(s, np.float64)
    return lib().or_percentile_sorted(_p(s), C.c_int64(len(s)), C.c_double(P))


class Quant:
    def __init__(self, min_f, max_f, scale_f, delta, p_l, p_h):
        self.min_f, self.max_f, self.scale_f = min_f, max_f, scale_f
        self.delta, self.p_l, self.p_h = delta, p_l, p_h


def train(x, sample, k_density=10, p_max=5.0, delta_override=float("nan"), eps=1e-6) -> Quant:
    x = _c(x, np.float32)
    sample = _c(sample, np.int32)
    d = x.shape[1]
    mn, mx, sc = (np.zeros(d, np.float32) for _ in range(3))
    meta = np.zeros(3, np.float64)
    st = lib().or_train(_p(x), C.c_int64(x.shape[0]), C.c_int32(d), _p(sample), C.c_int32(len(sample)),
                        C.c_int32(k_density), C.c_double(p_max), C.c_double(delta_override),
                        C.c_double(eps), _p(mn), _p(mx), _p(sc), _p(meta))
    if st:
        raise ValueError(f"or_train status {st}")
    return Quant(mn, mx, sc, float(meta[0]), float(meta[1]), float(meta[2]))


def d_pad_of(d: int) -> int:
    """Row stride of the code array used in the tests (16-byte multiple)."""
    return (d + 15) // 16 * 16


def encode(x, quant: Quant, d_pad=None):
    x = _c(x, np.float32)
    n, d = x.shape
    d_pad = d_pad_of(d) if d_pad is None else d_pad
    codes = np.zeros((n, d_pad), np.uint8)
    lib().or_encode(_p(x), C.c_int64(n), C.c_int32(d), _p(quant.min_f), _p(quant.scale_f), _p(codes),
                    C.c_int32(d_pad))
    return codes


# ------------------------------------------------------------------------------------------
# search phase
# ------------------------------------------------------------------------------------------

class Index:
    """Graph (from the host builder) + codes + fp32 base, as the oracle consumes them."""

    def __init__(self, x, codes, quant: Quant, graph, metric="l2"):
        self.x = _c(x, np.float32)
        self.codes = _c(codes, np.uint8)
        self.quant = quant
        self.g = graph
        self.metric = metric
        self.adj0 = _c(graph.adj0, np.int32)
        self.adj_upper = _c(graph.adj_upper, np.int32)
        self.upper_off = _c(graph.upper_off, np.int64)
        self.levels = _c(graph.levels, np.int32)
        s = _Index()
        s.n, s.d, s.d_pad = self.x.shape[0], self.x.shape[1], self.codes.shape[1]
        s.metric = 0 if metric == "l2" else 1
        s.codes, s.base = _p(self.codes), _p(self.x)
        s.min_f, s.scale_f = _p(quant.min_f), _p(quant.scale_f)
        s.max_level, s.entry_point = graph.max_level, graph.entry_point
        s.cap0, s.adj0 = self.adj0.shape[1], _p(self.adj0)
        s.capu = self.adj_upper.shape[1] if self.adj_upper.ndim == 2 else 1
        s.upper_off, s.adj_upper, s.levels = _p(self.upper_off), _p(self.adj_upper), _p(self.levels)
        self.s = s


def _params(k, ef, n_coarse, n_rerank, tau_gap, tau_ratio, early_term, assemble_mode, beam_form, traversal=0,
            tau_spread=float("inf")):
    p = _Params()
    p.tau_spread = tau_spread
    p.traversal = {"aqr": 0, "fp32": 1}[traversal] if isinstance(traversal, str) else int(traversal)
    p.k, p.ef, p.n_coarse, p.n_rerank = k, ef, n_coarse, n_rerank
    p.tau_gap, p.tau_ratio = tau_gap, tau_ratio
    p.early_term, p.assemble_mode, p.beam_form = int(early_term), assemble_mode, beam_form
    return p


def search(ix: Index, q, k, ef, n_coarse, n_rerank, tau_gap=0.010, tau_ratio=1.008, early_term=True,
           assemble_mode=0, beam_form=0, trace=False, exp_cap=4096, traversal="aqr", tau_spread=float("inf")):
    """traversal="aqr": Alg2.  traversal="fp32": the paper's baseline HNSW search
     on the same graph -- greedy + flag-form beam on exact fp32 distances in the canonical
    order R(L) (R22), result = the first k of W; coarse_dq then holds fp32 bits."""
    q = _c(q, np.float32)
    nq = q.shape[0]
    ids = np.zeros((nq, k), np.int32)
    dist = np.zeros((nq, k), np.float32)
    p = _params(k, ef, n_coarse, n_rerank, tau_gap, tau_ratio, early_term, assemble_mode, beam_form, traversal,
                tau_spread)
    tr = {}
    if trace:
        tr = dict(exp_ids=np.full((nq, exp_cap), -1, np.int32),
                  coarse_ids=np.full((nq, n_coarse), -1, np.int32),
                  coarse_dq=np.full((nq, n_coarse), -1, np.int32),
                  asym_ids=np.full((nq, n_coarse), -1, np.int32),
                  asym_d=np.full((nq, n_coarse), np.nan, np.float32),
                  exact_d=np.full((nq, n_coarse), np.nan, np.float32),
                  counters=np.zeros((nq, NCOUNT), np.int64),
                  upper_end=np.full((nq, max(ix.g.max_level, 1)), -1, np.int32))
    g = tr.get
    st = lib().or_search(C.byref(ix.s), _p(q), C.c_int64(nq), C.byref(p), _p(ids), _p(dist),
                         C.c_int32(exp_cap), _p(g("exp_ids")), _p(g("coarse_ids")), _p(g("coarse_dq")),
                         _p(g("asym_ids")), _p(g("asym_d")), _p(g("exact_d")), _p(g("counters")),
                         C.c_int32(max(ix.g.max_level, 1)), _p(g("upper_end")))
    if st:
        raise ValueError(f"or_search status {st}")
    if trace:
        return ids, dist, tr
    return ids, dist


def rerank(ix: Index, q, cand, k, n_rerank, tau_gap=0.010, tau_ratio=1.008, early_term=True,
           assemble_mode=0, tau_spread=float("inf")):
    q = _c(q, np.float32)
    cand = _c(cand, np.int32)
    nq = q.shape[0]
    ids = np.zeros((nq, k), np.int32)
    dist = np.zeros((nq, k), np.float32)
    p = _params(k, cand.shape[1], cand.shape[1], n_rerank, tau_gap, tau_ratio, early_term, assemble_mode, 0,
                tau_spread=tau_spread)
    st = lib().or_rerank(C.byref(ix.s), _p(q), C.c_int64(nq), _p(cand), C.c_int32(cand.shape[1]),
                         C.byref(p), _p(ids), _p(dist))
    if st:
        raise ValueError(f"or_rerank status {st}")
    return ids, dist


def merge_topk(dist, ids, k):
    """dist/ids: [S, nq, k_in] per-shard sorted lists (global ids) -> [nq, k]."""
    dist = _c(dist, np.float32)
    ids = _c(ids, np.int32)
    S, nq, kin = ids.shape
    assert kin == k
    od = np.zeros((nq, k), np.float32)
    oi = np.zeros((nq, k), np.int32)
    st = lib().or_merge_topk(_p(dist), _p(ids), C.c_int32(S), C.c_int64(nq), C.c_int32(k), _p(od), _p(oi))
    if st:
        raise ValueError(f"or_merge_topk status {st}")
    return od, oi


def bruteforce(x, q, k, metric="l2"):
    x = _c(x, np.float32)
    q = _c(q, np.float32)
    ids = np.zeros((q.shape[0], k), np.int32)
    d = np.zeros((q.shape[0], k), np.float64)
    lib().or_bruteforce(_p(x), C.c_int64(x.shape[0]), C.c_int32(x.shape[1]), _p(q), C.c_int64(q.shape[0]),
                        C.c_int32(k), C.c_int32(0 if metric == "l2" else 1), _p(ids), _p(d))
    return ids, d


def bruteforce_dq(codes, d, qcodes, k):
    codes = _c(codes, np.uint8)
    qcodes = _c(qcodes, np.uint8)
    ids = np.zeros((qcodes.shape[0], k), np.int32)
    dd = np.zeros((qcodes.shape[0], k), np.int32)
    lib().or_bruteforce_dq(_p(codes), C.c_int64(codes.shape[0]), C.c_int32(d), C.c_int32(codes.shape[1]),
                           _p(qcodes), C.c_int64(qcodes.shape[0]), C.c_int32(k), _p(ids), _p(dd))
    return ids, dd


def ef_mapping(ef: int, k: int, m_ef: int = 3, n_rerank_preset: int = 28):
    """DESIGN.md R13: BJ's "ef" is ef_search; preset "0.97+" of Table 3:
    N_c = max(k, floor(ef/m_ef)), N_rerank = min(max(k, 28), N_c)."""
    n_c = max(k, ef // m_ef)
    n_c = min(n_c, ef) if ef >= k else k
    return dict(ef=max(ef, n_c), n_coarse=n_c, n_rerank=min(max(k, n_rerank_preset), n_c))


# ------------------------------------------------------------------------------------------
# single-pair hooks (pin tests)
# ------------------------------------------------------------------------------------------

def dist_quantized(qc, xc):
    qc = _c(qc, np.uint8)
    xc = _c(xc, np.uint8)
    return int(lib().or_dist_quantized(_p(qc), _p(xc), C.c_int32(len(qc))))


def dist_asym(q, xc, min_f, scale_f, metric="l2"):
    L = lib()
    L.or_dist_asym.restype = C.c_float
    q, xc = _c(q, np.float32), _c(xc, np.uint8)
    mn, sc = _c(min_f, np.float32), _c(scale_f, np.float32)
    return float(L.or_dist_asym(_p(q), _p(xc), _p(mn), _p(sc), C.c_int32(len(q)), C.c_int32(0 if metric == "l2" else 1)))


def dist_fp_RL(q, x, metric="l2"):
    """Exact fp32 distance in the canonical order R(L) of the FP32-HNSW baseline (R22)."""
    L = lib()
    L.or_dist_fp_RL.restype = C.c_float
    q = _c(q, np.float32)
    x = _c(x, np.float32)
    return float(L.or_dist_fp_RL(_p(q), _p(x), C.c_int32(len(q)), C.c_int32(0 if metric == "l2" else 1)))


def dist_exact(q, x, metric="l2"):
    L = lib()
    L.or_dist_exact.restype = C.c_float
    q, x = _c(q, np.float32), _c(x, np.float32)
    return float(L.or_dist_exact(_p(q), _p(x), C.c_int32(len(q)), C.c_int32(0 if metric == "l2" else 1)))


def decode(code, scale, mn):
    L = lib()
    L.or_decode.restype = C.c_float
    return float(L.or_decode(C.c_uint8(code), C.c_float(scale), C.c_float(mn)))


# ------------------------------------------------------------------------------------------
# graph construction (Alg1 l.16-22; the oracle of the GPU index build, R28)
# ------------------------------------------------------------------------------------------
def build_levels(u, M):
    """Node levels floor(-ln(u) / ln(M)), capped at 30, from uniform draws u in (0, 1]."""
    u = _c(u, np.float64)
    lv = np.zeros(len(u), np.int32)
    lib().or_build_levels(_p(u), C.c_int64(len(u)), C.c_int32(M), _p(lv))
    return lv


def build_graph(codes, d, M, efc, level_u, flags=1, batch_div=32):
    """HNSW insertion over the codes [n, d_pad] in the wave order of DESIGN.md R28 ->
    (levels, upper_off, adj0 [n, 2M], adj_upper [rows, M], entry_point, max_level)."""
    codes = _c(codes, np.uint8)
    n, d_pad = codes.shape
    levels = build_levels(level_u, M)
    upper_off = np.zeros(n, np.int64)
    rows = int(lib().or_build_upper_rows(_p(levels), C.c_int64(n), _p(upper_off)))
    adj0 = np.zeros((n, 2 * M), np.int32)
    adj_upper = np.zeros((max(rows, 1), M), np.int32)
    em = np.zeros(2, np.int32)
    L = lib()
    L.or_build_upper_rows.restype = C.c_int64
    st = L.or_build_graph(_p(codes), C.c_int64(n), C.c_int32(d), C.c_int32(d_pad), _p(levels), _p(upper_off),
                          C.c_int32(M), C.c_int32(efc), C.c_int32(flags), C.c_int32(batch_div), _p(adj0),
                          _p(adj_upper), _p(em))
    if st:
        raise ValueError(f"or_build_graph status {st}")
    return levels, upper_off, adj0, adj_upper[:rows], int(em[0]), int(em[1])
