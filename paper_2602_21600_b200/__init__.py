"""aqr-b200: B200-native AQR-HNSW batched k-NN search (arXiv 2602.21600).

Thin Python binding of the C ABI in include/aqr.h (libaqr.so, sm_100a).  Argument
marshalling only: every step of the hot path runs in the CUDA kernels behind the ABI.
PyTorch supplies device memory and streams.  There is NO CPU fallback: if libaqr.so is
missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from . import build as _build

_PKG = os.path.dirname(os.path.abspath(__file__))

AQR_L2, AQR_IP = 0, 1
NCOUNT = 15
COUNTER_NAMES = ["expansions", "deg_sum", "evals", "upper_exp", "upper_deg_sum", "upper_evals", "n_coarse",
                 "depth", "early_term", "n_asym", "hash_fail", "below_thr", "w_inserts", "reserved13", "reserved14"]


class AqrError(RuntimeError):
    pass


class QuantParams(C.Structure):
    _fields_ = [("d", C.c_int32), ("d_pad", C.c_int32), ("min_j", C.c_void_p), ("max_j", C.c_void_p),
                ("scale_j", C.c_void_p), ("delta", C.c_double), ("p_low", C.c_double), ("p_high", C.c_double)]


class TrainCfg(C.Structure):
    _fields_ = [("sample_idx", C.c_void_p), ("n_sample", C.c_int32), ("k_density", C.c_int32),
                ("p_max", C.c_double), ("eps", C.c_double), ("delta_override", C.c_double),
                ("rho_out", C.c_void_p)]


class IndexDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("metric", C.c_int32), ("id_base", C.c_int64),
                ("codes", C.c_void_p), ("d_pad", C.c_int32), ("base", C.c_void_p), ("ld_base", C.c_int64),
                ("min_j", C.c_void_p), ("scale_j", C.c_void_p), ("M", C.c_int32), ("max_level", C.c_int32),
                ("entry_point", C.c_int32), ("adj0", C.c_void_p), ("upper_off", C.c_void_p),
                ("adj_upper", C.c_void_p), ("upper_rows", C.c_int64), ("layout", C.c_int32)]


class SearchParams(C.Structure):
    _fields_ = [("k", C.c_int32), ("ef", C.c_int32), ("n_coarse", C.c_int32), ("n_rerank", C.c_int32),
                ("tau_gap", C.c_double), ("tau_ratio", C.c_double), ("early_term", C.c_int32),
                ("assemble_mode", C.c_int32), ("visited_bits", C.c_int32), ("warps_per_block", C.c_int32),
                ("traversal", C.c_int32), ("tau_spread", C.c_double), ("warps_per_query", C.c_int32)]


class Debug(C.Structure):
    _fields_ = [("exp_cap", C.c_int32), ("exp_ids", C.c_void_p), ("coarse_ids", C.c_void_p),
                ("coarse_dq", C.c_void_p), ("asym_ids", C.c_void_p), ("asym_d", C.c_void_p),
                ("exact_d", C.c_void_p), ("counters", C.c_void_p), ("totals", C.c_void_p),
                ("t_ns", C.c_void_p)]


LAYOUTS = {"auto": 0, "gather": 1, "inline": 2}
EXPORTS = ["aqr_encode", "aqr_upload_index", "aqr_index_free", "aqr_index_device_bytes", "aqr_index_layout",
           "aqr_search_workspace_size",
           "aqr_search", "aqr_search_plan", "aqr_rerank", "aqr_merge_topk", "aqr_build_graph", "aqr_last_error", "aqr_version"]

_lib = None


def lib_path() -> str:
    """libaqr.so, or libaqr_<v>.so when AQR_LIB_VARIANT=v (a test build, e.g. the bounds-checked one)."""
    v = os.environ.get("AQR_LIB_VARIANT")
    return os.path.join(_PKG, f"libaqr_{v}.so") if v else _build.LIB_AQR


def lib():
    """Load libaqr.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise AqrError(f"libaqr.so not built ({path}); run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(path)
        L.aqr_last_error.restype = C.c_char_p
        L.aqr_version.restype = C.c_char_p
        L.aqr_index_device_bytes.restype = C.c_size_t
        L.aqr_search_workspace_size.restype = C.c_size_t
        L.aqr_index_layout.restype = C.c_int32
        for f in ["aqr_encode", "aqr_upload_index", "aqr_search", "aqr_rerank", "aqr_merge_topk", "aqr_build_graph"]:
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(st: int, what: str):
    if st != 0:
        raise AqrError(f"{what} failed (status {st}): {lib().aqr_last_error().decode()}")


def _torch():
    import torch
    return torch


def _dev(t, dtype, name):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise AqrError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise AqrError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise AqrError(f"{name} must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def d_pad_of(d: int) -> int:
    return (d + 15) // 16 * 16


# --------------------------------------------------------------------------------------
# aqr_encode
# --------------------------------------------------------------------------------------

class Quantizer:
    """Trained per-dimension quantizer (device tensors min_j / max_j / scale_j)."""

    def __init__(self, d, device):
        torch = _torch()
        self.d = d
        self.d_pad = d_pad_of(d)
        self.min_j = torch.zeros(d, dtype=torch.float32, device=device)
        self.max_j = torch.zeros(d, dtype=torch.float32, device=device)
        self.scale_j = torch.ones(d, dtype=torch.float32, device=device)
        self.delta = self.p_low = self.p_high = float("nan")
        self.rho = None

    def _struct(self):
        qp = QuantParams()
        qp.d, qp.d_pad = self.d, self.d_pad
        qp.min_j, qp.max_j, qp.scale_j = self.min_j.data_ptr(), self.max_j.data_ptr(), self.scale_j.data_ptr()
        qp.delta, qp.p_low, qp.p_high = self.delta, self.p_low, self.p_high
        return qp


def encode(x, quant: Quantizer | None = None, sample_idx=None, k_density=10, p_max=5.0, eps=1e-6,
           delta_override=None, want_rho=False, stream=None):
    """aqr_encode: train (if `quant` is None) and encode x [n, d] fp32 CUDA -> (codes [n, d_pad] u8, quantizer)."""
    torch = _torch()
    px = _dev(x, torch.float32, "x")
    n, d = x.shape
    train = None
    if quant is None:
        quant = Quantizer(d, x.device)
        if sample_idx is None:
            raise AqrError("training needs sample_idx (sorted int32 CUDA tensor)")
        psi = _dev(sample_idx, torch.int32, "sample_idx")
        train = TrainCfg()
        train.sample_idx, train.n_sample, train.k_density = psi.value, sample_idx.numel(), k_density
        train.p_max, train.eps = p_max, eps
        train.delta_override = float("nan") if delta_override is None else float(delta_override)
        if want_rho:
            quant.rho = torch.zeros(sample_idx.numel(), dtype=torch.float64, device=x.device)
            train.rho_out = quant.rho.data_ptr()
    codes = torch.empty((n, quant.d_pad), dtype=torch.uint8, device=x.device)
    qp = quant._struct()
    st = lib().aqr_encode(px, C.c_int64(n), C.c_int32(d), C.c_int64(d), C.byref(train) if train else None,
                          C.byref(qp), C.c_void_p(codes.data_ptr()), _stream(stream))
    _check(st, "aqr_encode")
    if train is not None:
        quant.delta, quant.p_low, quant.p_high = qp.delta, qp.p_low, qp.p_high
    return codes, quant


# --------------------------------------------------------------------------------------
# aqr_upload_index
# --------------------------------------------------------------------------------------

class Index:
    """Library-owned device index (aqr_index*).  Freed with .free() or on garbage collection."""

    def __init__(self, handle, n, d, k_metric, id_base, M):
        self._h = handle
        self.n, self.d, self.metric, self.id_base, self.M = n, d, k_metric, id_base, M

    @property
    def handle(self):
        if self._h is None:
            raise AqrError("index already freed")
        return self._h

    @property
    def layout(self) -> str:
        return {1: "gather", 2: "inline"}.get(int(lib().aqr_index_layout(self.handle)), "?")

    def device_bytes(self) -> int:
        return int(lib().aqr_index_device_bytes(self.handle))

    def free(self):
        if self._h is not None:
            lib().aqr_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def upload_index(codes, base, quant: Quantizer, graph, metric="l2", id_base=0, layout="auto", stream=None) -> Index:
    """aqr_upload_index: codes [n, d_pad] u8 CUDA, base [n, d] fp32 CUDA, graph (host arrays)."""
    torch = _torch()
    _dev(codes, torch.uint8, "codes")
    _dev(base, torch.float32, "base")
    n, d = base.shape
    adj0 = np.ascontiguousarray(graph.adj0, dtype=np.int32)
    upper_off = np.ascontiguousarray(graph.upper_off, dtype=np.int64)
    adj_upper = np.ascontiguousarray(graph.adj_upper, dtype=np.int32)
    D = IndexDesc()
    D.n, D.d, D.metric, D.id_base = n, d, AQR_L2 if metric == "l2" else AQR_IP, int(id_base)
    D.codes, D.d_pad = codes.data_ptr(), codes.shape[1]
    D.base, D.ld_base = base.data_ptr(), d
    D.min_j, D.scale_j = quant.min_j.data_ptr(), quant.scale_j.data_ptr()
    D.M, D.max_level, D.entry_point = int(graph.M), int(graph.max_level), int(graph.entry_point)
    D.adj0 = adj0.ctypes.data
    D.upper_off = upper_off.ctypes.data
    D.adj_upper = adj_upper.ctypes.data if adj_upper.size else None
    D.upper_rows = adj_upper.shape[0] if adj_upper.size else 0
    D.layout = LAYOUTS[layout]
    h = C.c_void_p()
    st = lib().aqr_upload_index(C.byref(D), C.byref(h), _stream(stream))
    _check(st, "aqr_upload_index")
    return Index(h, n, d, metric, id_base, graph.M)


# --------------------------------------------------------------------------------------
# aqr_search / aqr_rerank / aqr_merge_topk
# --------------------------------------------------------------------------------------

def ef_mapping(ef: int, k: int, m_ef: int = 3, n_rerank_preset: int = 28):
    """DESIGN.md R13 (Table 3 preset "0.97+"): N_c = max(k, ef // m_ef),
    N_rerank = min(max(k, 28), N_c); ef_search = max(ef, N_c)."""
    n_c = max(k, ef // m_ef)
    return dict(ef=max(ef, n_c), n_coarse=n_c, n_rerank=min(max(k, n_rerank_preset), n_c))


TRAVERSALS = {"aqr": 0, "fp32": 1}


def make_params(k, ef, n_coarse, n_rerank, tau_gap=0.010, tau_ratio=1.008, early_term=True, assemble_mode=0,
                visited_bits=0, warps_per_block=0, traversal="aqr", tau_spread=math.inf,
                warps_per_query=0) -> SearchParams:
    """warps_per_query: 0 auto, 1 one warp per query, 4 one cooperative CTA of 4 warps (include/aqr.h)."""
    p = SearchParams()
    p.warps_per_query = warps_per_query
    p.tau_spread = tau_spread
    p.traversal = TRAVERSALS[traversal]
    p.k, p.ef, p.n_coarse, p.n_rerank = k, ef, n_coarse, n_rerank
    p.tau_gap, p.tau_ratio = tau_gap, tau_ratio
    p.early_term, p.assemble_mode = int(bool(early_term)), assemble_mode
    p.visited_bits, p.warps_per_block = visited_bits, warps_per_block
    return p


def search_plan(index: Index, nq: int, params: SearchParams) -> int:
    """Warps per query aqr_search would use for this launch (1 or 4; aqr_search_plan)."""
    g = C.c_int32(0)
    _check(lib().aqr_search_plan(index.handle, C.c_int64(nq), C.byref(params), C.byref(g)), "aqr_search_plan")
    return int(g.value)


class Searcher:
    """Pre-allocated outputs + workspace for repeated aqr_search calls (bench loop)."""

    def __init__(self, index: Index, nq: int, params: SearchParams, device="cuda"):
        torch = _torch()
        self.index, self.nq, self.params = index, nq, params
        self.ids = torch.empty((nq, params.k), dtype=torch.int32, device=device)
        self.dist = torch.empty((nq, params.k), dtype=torch.float32, device=device)
        ws = int(lib().aqr_search_workspace_size(index.handle, C.c_int64(nq), C.byref(params)))
        self.ws = torch.empty(ws, dtype=torch.uint8, device=device)
        self.totals = torch.zeros(NCOUNT, dtype=torch.int64, device=device)
        self._dbg = Debug()
        self._dbg.totals = self.totals.data_ptr()
        self._tdbg = None
        self.t_ns = None

    def run(self, q, stream=None, stats=False, timing=False, out=None):
        """timing=True: per-query [start, end] %globaltimer ns into self.t_ns [nq, 2] (no counters).
        out=(ids_ptr, dist_ptr): raw device addresses of [q.shape[0] x k] int32 / fp32 outputs written
        instead of self.ids / self.dist (a peer GPU's gather buffer, PeerExchange.dest)."""
        torch = _torch()
        pq = _dev(q, torch.float32, "q")
        if q.dim() != 2 or q.shape[1] != self.index.d:
            raise AqrError(f"q must be [nq, {self.index.d}], got {tuple(q.shape)}")
        if q.shape[0] > self.nq:
            raise AqrError(f"batch of {q.shape[0]} queries exceeds this Searcher's {self.nq} (outputs are sized for it)")
        dbg = None
        if stats:
            dbg = C.byref(self._dbg)
        elif timing:
            if self.t_ns is None:
                self.t_ns = torch.zeros((self.nq, 2), dtype=torch.int64, device=self.ids.device)
                self._tdbg = Debug()
                self._tdbg.t_ns = self.t_ns.data_ptr()
            dbg = C.byref(self._tdbg)
        o_ids, o_dist = (self.ids.data_ptr(), self.dist.data_ptr()) if out is None else (int(out[0]), int(out[1]))
        st = lib().aqr_search(self.index.handle, pq, C.c_int64(q.shape[0]), C.c_int64(q.shape[1]),
                              C.byref(self.params), C.c_void_p(o_ids), C.c_void_p(o_dist), dbg,
                              C.c_void_p(self.ws.data_ptr()), C.c_size_t(self.ws.numel()), _stream(stream))
        _check(st, "aqr_search")
        return (self.ids, self.dist) if out is None else None


def search(index: Index, q, k, ef, n_coarse, n_rerank, tau_gap=0.010, tau_ratio=1.008, early_term=True,
           assemble_mode=0, visited_bits=0, warps_per_block=0, trace=False, exp_cap=4096, stream=None,
           traversal="aqr", tau_spread=math.inf, warps_per_query=0):
    """aqr_search on q [nq, d] fp32 CUDA -> (ids [nq, k] int32, dist [nq, k] fp32[, trace dict])."""
    torch = _torch()
    pq = _dev(q, torch.float32, "q")
    if q.dim() != 2 or q.shape[1] != index.d:
        raise AqrError(f"q must be [nq, {index.d}], got {tuple(q.shape)}")
    nq = q.shape[0]
    p = make_params(k, ef, n_coarse, n_rerank, tau_gap, tau_ratio, early_term, assemble_mode, visited_bits,
                    warps_per_block, traversal, tau_spread, warps_per_query)
    dev = q.device
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dist = torch.empty((nq, k), dtype=torch.float32, device=dev)
    ws = torch.empty(int(lib().aqr_search_workspace_size(index.handle, C.c_int64(nq), C.byref(p))),
                     dtype=torch.uint8, device=dev)
    dbg = None
    tr = None
    if trace:
        tr = dict(exp_ids=torch.full((nq, exp_cap), -1, dtype=torch.int32, device=dev),
                  coarse_ids=torch.full((nq, n_coarse), -1, dtype=torch.int32, device=dev),
                  coarse_dq=torch.full((nq, n_coarse), -1, dtype=torch.int32, device=dev),
                  asym_ids=torch.full((nq, n_coarse), -1, dtype=torch.int32, device=dev),
                  asym_d=torch.full((nq, n_coarse), float("nan"), dtype=torch.float32, device=dev),
                  exact_d=torch.full((nq, n_coarse), float("nan"), dtype=torch.float32, device=dev),
                  counters=torch.zeros((nq, NCOUNT), dtype=torch.int64, device=dev),
                  totals=torch.zeros(NCOUNT, dtype=torch.int64, device=dev))
        dbg = Debug()
        dbg.exp_cap = exp_cap
        for f in ["exp_ids", "coarse_ids", "coarse_dq", "asym_ids", "asym_d", "exact_d", "counters", "totals"]:
            setattr(dbg, f, tr[f].data_ptr())
    st = lib().aqr_search(index.handle, pq, C.c_int64(nq), C.c_int64(q.shape[1]), C.byref(p),
                          C.c_void_p(ids.data_ptr()), C.c_void_p(dist.data_ptr()),
                          C.byref(dbg) if dbg is not None else None, C.c_void_p(ws.data_ptr()),
                          C.c_size_t(ws.numel()), _stream(stream))
    _check(st, "aqr_search")
    if trace:
        return ids, dist, tr
    return ids, dist


def rerank(index: Index, q, cand_ids, k, n_rerank, tau_gap=0.010, tau_ratio=1.008, early_term=True,
           assemble_mode=0, stream=None, tau_spread=math.inf):
    """aqr_rerank: Stages 2 / ET / 3 / assembly on cand_ids [nq, n_cand] int32 CUDA (sorted by (d^q, id))."""
    torch = _torch()
    pq = _dev(q, torch.float32, "q")
    pc = _dev(cand_ids, torch.int32, "cand_ids")
    nq, nc = cand_ids.shape
    p = make_params(k, nc, nc, n_rerank, tau_gap, tau_ratio, early_term, assemble_mode, tau_spread=tau_spread)
    ids = torch.empty((nq, k), dtype=torch.int32, device=q.device)
    dist = torch.empty((nq, k), dtype=torch.float32, device=q.device)
    st = lib().aqr_rerank(index.handle, pq, C.c_int64(nq), C.c_int64(q.shape[1]), pc, C.c_int32(nc), C.byref(p),
                          C.c_void_p(ids.data_ptr()), C.c_void_p(dist.data_ptr()), _stream(stream))
    _check(st, "aqr_rerank")
    return ids, dist


def merge_topk(dist, ids, k=None, stream=None):
    """aqr_merge_topk: dist/ids [S, nq, k] CUDA (rows sorted by (dist, id)) -> (dist [nq, k], ids [nq, k])."""
    torch = _torch()
    pd = _dev(dist, torch.float32, "dist")
    pi = _dev(ids, torch.int32, "ids")
    S, nq, kk = ids.shape
    k = kk if k is None else k
    if k != kk:
        raise AqrError("k must equal the list length")
    od = torch.empty((nq, k), dtype=torch.float32, device=dist.device)
    oi = torch.empty((nq, k), dtype=torch.int32, device=dist.device)
    st = lib().aqr_merge_topk(pd, pi, C.c_int32(S), C.c_int64(nq), C.c_int32(k), C.c_void_p(od.data_ptr()),
                              C.c_void_p(oi.data_ptr()), _stream(stream))
    _check(st, "aqr_merge_topk")
    return od, oi


# --------------------------------------------------------------------------------------
# peer-memory exchange (include/aqr.h "Peer-memory exchange"; parallel.PeerExchange drives it)
# --------------------------------------------------------------------------------------
PEER_HANDLE_BYTES = 64
MAX_PEERS = 8


class PeerBuffer:
    """Device memory from aqr_peer_alloc (owner) or a peer's allocation mapped by aqr_peer_open."""

    def __init__(self, ptr: int, nbytes: int, owner: bool, handle: bytes = b""):
        self.ptr, self.nbytes, self.owner, self.handle = ptr, nbytes, owner, handle

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False), "version": 2}

    def tensor(self, dtype, shape, offset=0):
        """A torch view of [offset, offset + prod(shape) x itemsize) -- LOCAL (owner) buffers only."""
        torch = _torch()
        if not self.owner:
            raise AqrError("tensor views are for the local buffer; peers are addressed by pointer")
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        if offset < 0 or offset + n > self.nbytes:
            raise AqrError("view outside the buffer")
        raw = torch.as_tensor(self, device="cuda")
        return raw[offset:offset + n].view(dtype).view(*shape)

    def close(self):
        if self.ptr:
            fn = lib().aqr_peer_free if self.owner else lib().aqr_peer_close
            _check(fn(C.c_void_p(self.ptr)), "aqr_peer_free" if self.owner else "aqr_peer_close")
            self.ptr = 0


def peer_alloc(nbytes: int) -> PeerBuffer:
    p = C.c_void_p()
    h = (C.c_uint8 * PEER_HANDLE_BYTES)()
    _check(lib().aqr_peer_alloc(C.c_size_t(nbytes), C.byref(p), h), "aqr_peer_alloc")
    return PeerBuffer(int(p.value), nbytes, True, bytes(h))


def peer_open(handle: bytes, nbytes: int) -> PeerBuffer:
    if len(handle) != PEER_HANDLE_BYTES:
        raise AqrError("bad peer handle")
    p = C.c_void_p()
    h = (C.c_uint8 * PEER_HANDLE_BYTES).from_buffer_copy(handle)
    _check(lib().aqr_peer_open(h, C.byref(p)), "aqr_peer_open")
    return PeerBuffer(int(p.value), nbytes, False)


def peer_signal(flag_ptrs, slot: int, value: int, stream=None):
    """aqr_peer_signal: flag_ptrs = device addresses (ints) of every rank's flag array."""
    arr = (C.c_void_p * len(flag_ptrs))(*[C.c_void_p(int(v)) for v in flag_ptrs])
    _check(lib().aqr_peer_signal(arr, C.c_int32(len(flag_ptrs)), C.c_int32(slot), C.c_uint64(value), _stream(stream)),
           "aqr_peer_signal")


def peer_wait(flags_ptr: int, n: int, value: int, timeout_ns: int, status=None, stream=None):
    """aqr_peer_wait on the local flag array; status: a zeroed CUDA int32 tensor (or None)."""
    sp = C.c_void_p(status.data_ptr()) if status is not None else C.c_void_p(0)
    _check(lib().aqr_peer_wait(C.c_void_p(int(flags_ptr)), C.c_int32(n), C.c_uint64(value), C.c_uint64(timeout_ns), sp,
                               _stream(stream)), "aqr_peer_wait")


from .graph import Graph, build_hnsw, build_hnsw_gpu, adapt_params  # noqa: E402,F401
