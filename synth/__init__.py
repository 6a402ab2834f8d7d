"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the AQR-HNSW method (no density, no quantizer, no
distance, no search).  It only draws random numbers: base vectors, queries, the density
sample indices ("compute densities for a sample of n_s = min(5000, n) points") and
the HNSW level draws ("level = floor(-ln(draw) * mL)" -- the draws only; the
builder applies the formula).  Random numbers the method consumes are passed to both
sides as inputs (task rule 3).

Workloads follow BASELINE.json `configs` C1..C5 (restated in SURVEY.md 8(d)); the
paper's real datasets (SIFT-1M, GloVe, GIST-1M) are not available and these
distributions stand in for them.

Streams: numpy default_rng(SeedSequence([seed, cfg_id, stream])), stream 0 = base,
1 = queries, 2 = density sample, 3 = supplementary query stream, 4 = level draws.
"""
from __future__ import annotations

import dataclasses
import hashlib

import numpy as np

CFG_IDS = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5, "tiny": 90, "grid": 91}


def _rng(seed: int, cfg: str, stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), CFG_IDS.get(cfg, 99), int(stream)]))


@dataclasses.dataclass
class Workload:
    name: str
    x: np.ndarray          # [n, d] float32 base vectors
    q: np.ndarray          # [nq, d] float32 queries
    metric: str            # "l2" | "ip"
    M0: int                # Alg1 line 1 input M_0
    efc0: int              # Alg1 line 1 input ef_0^construction
    ef: int                # BJ "ef" (ef_search)
    k: int
    seed: int = 0


# ---------------------------------------------------------------------------------
# distributions (BASELINE.json configs; unspecified parameters per SURVEY 8(d) <p>)
# ---------------------------------------------------------------------------------

def _gmm(rng, n, d, n_comp, sig_lo, sig_hi, centres=None, sigmas=None, chunk=1 << 20):
    if centres is None:
        centres = rng.uniform(-1.0, 1.0, size=(n_comp, d))
    if sigmas is None:
        sigmas = np.exp(rng.uniform(np.log(sig_lo), np.log(sig_hi), size=n_comp))
    out = np.empty((n, d), dtype=np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        comp = rng.integers(0, n_comp, size=e - s)
        z = rng.standard_normal(size=(e - s, d))
        out[s:e] = (centres[comp] + sigmas[comp][:, None] * z).astype(np.float32)
    return out


def _mixture_params(seed, cfg, d, n_comp, sig_lo, sig_hi):
    # the mixture itself (centres, sigmas) is drawn once from stream 5 so that base
    # vectors and queries come from the SAME distribution (BJ: "queries from the same mixture")
    r = _rng(seed, cfg, 5)
    centres = r.uniform(-1.0, 1.0, size=(n_comp, d))
    sigmas = np.exp(r.uniform(np.log(sig_lo), np.log(sig_hi), size=n_comp))
    return centres, sigmas


def gen_c1(n=10_000, nq=100, seed=0, d=128):
    c, s = _mixture_params(seed, "C1", d, 16, 0.05, 1.0)
    x = _gmm(_rng(seed, "C1", 0), n, d, 16, 0, 0, c, s)
    q = _gmm(_rng(seed, "C1", 1), nq, d, 16, 0, 0, c, s)
    return Workload("C1", x, q, "l2", M0=16, efc0=100, ef=64, k=10, seed=seed)


def _gamma_int(rng, n, d, theta=40.0, chunk=1 << 18):
    out = np.empty((n, d), dtype=np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        g = rng.gamma(0.5, 1.0, size=(e - s, d)) * theta
        out[s:e] = np.rint(np.clip(g, 0.0, 218.0)).astype(np.float32)
    return out


def gen_c2(n=1_000_000, nq=10_000, seed=0, d=128):
    x = _gamma_int(_rng(seed, "C2", 0), n, d)
    q = _gamma_int(_rng(seed, "C2", 1), nq, d)
    return Workload("C2", x, q, "l2", M0=16, efc0=200, ef=128, k=10, seed=seed)


def _aniso_unit(rng, n, d, chunk=1 << 18):
    v = (1.0 + np.arange(d)) ** -0.7
    sd = np.sqrt(v)
    out = np.empty((n, d), dtype=np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        y = rng.standard_normal(size=(e - s, d)) * sd
        y /= np.linalg.norm(y, axis=1, keepdims=True)
        out[s:e] = y.astype(np.float32)
    return out


def gen_c3(n=1_180_000, nq=10_000, seed=0, d=100):
    x = _aniso_unit(_rng(seed, "C3", 0), n, d)
    q = _aniso_unit(_rng(seed, "C3", 1), nq, d)
    return Workload("C3", x, q, "ip", M0=24, efc0=200, ef=128, k=10, seed=seed)


def gen_c4(n=1_000_000, nq=1_000, seed=0, d=960):
    c, s = _mixture_params(seed, "C4", d, 64, 0.02, 0.5)
    x = np.abs(_gmm(_rng(seed, "C4", 0), n, d, 64, 0, 0, c, s, chunk=1 << 16))
    q = np.abs(_gmm(_rng(seed, "C4", 1), nq, d, 64, 0, 0, c, s, chunk=1 << 16))
    return Workload("C4", x, q, "l2", M0=32, efc0=200, ef=128, k=10, seed=seed)


def gen_c5_shard(shard: int, n_shard=1_250_000, seed=0, d=96):
    """Rows [n_shard*shard, n_shard*(shard+1)) of the 10M C5 base (generated per shard)."""
    c, s = _mixture_params(seed, "C5", d, 1024, 0.01, 1.0)
    r = np.random.default_rng(np.random.SeedSequence([seed, CFG_IDS["C5"], 0, shard]))
    return _gmm(r, n_shard, d, 1024, 0, 0, c, s)


def gen_c5_queries(nq=10_000, seed=0, d=96):
    c, s = _mixture_params(seed, "C5", d, 1024, 0.01, 1.0)
    return _gmm(_rng(seed, "C5", 1), nq, d, 1024, 0, 0, c, s)


def gen_c5(n_shard=1_250_000, n_shards=8, nq=10_000, seed=0):
    x = np.concatenate([gen_c5_shard(r, n_shard, seed) for r in range(n_shards)])
    return Workload("C5", x, gen_c5_queries(nq, seed), "l2", M0=32, efc0=200, ef=128, k=100, seed=seed)


def gen_config(name: str, scale: float = 1.0, seed: int = 0, nq: int | None = None) -> Workload:
    """Generate config `name`; `scale` < 1 gives a row-prefix-sized slice (same distribution)."""
    full = {"C1": (10_000, 100), "C2": (1_000_000, 10_000), "C3": (1_180_000, 10_000),
            "C4": (1_000_000, 1_000), "C5": (1_250_000, 10_000)}[name]
    n = max(1, int(round(full[0] * scale)))
    nq = full[1] if nq is None else nq
    if name == "C1":
        return gen_c1(n, nq, seed)
    if name == "C2":
        return gen_c2(n, nq, seed)
    if name == "C3":
        return gen_c3(n, nq, seed)
    if name == "C4":
        return gen_c4(n, nq, seed)
    w = Workload("C5", gen_c5_shard(0, n, seed), gen_c5_queries(nq, seed), "l2", 32, 200, 128, 100, seed)
    return w


def gen_query_stream(name: str, nq: int, seed: int = 0) -> np.ndarray:
    """Supplementary query stream (stream 3): fresh queries from the config's
    distribution, for steady-state throughput where the config's own query set under-fills the
    GPU (C1: 100 queries, C4: 1k).  Recall is always measured on the config's query set."""
    r = _rng(seed, name, 3)
    if name == "C1":
        c, s = _mixture_params(seed, "C1", 128, 16, 0.05, 1.0)
        return _gmm(r, nq, 128, 16, 0, 0, c, s)
    if name == "C2":
        return _gamma_int(r, nq, 128)
    if name == "C3":
        return _aniso_unit(r, nq, 100)
    if name == "C4":
        c, s = _mixture_params(seed, "C4", 960, 64, 0.02, 0.5)
        return np.abs(_gmm(r, nq, 960, 64, 0, 0, c, s, chunk=1 << 16))
    c, s = _mixture_params(seed, "C5", 96, 1024, 0.01, 1.0)
    return _gmm(r, nq, 96, 1024, 0, 0, c, s)


# ---------------------------------------------------------------------------------
# small fixtures
# ---------------------------------------------------------------------------------

def gen_tiny(n=600, d=7, nq=20, seed=0, metric="l2", n_comp=4):
    """Small clustered fixture with an arbitrary d (exercises tails: d = 7, 100, 960 ...)."""
    r = _rng(seed, "tiny", 0)
    centres = r.uniform(-1, 1, size=(n_comp, d))
    sig = np.exp(r.uniform(np.log(0.05), np.log(0.6), size=n_comp))
    x = _gmm(r, n, d, n_comp, 0, 0, centres, sig)
    q = _gmm(_rng(seed, "tiny", 1), nq, d, n_comp, 0, 0, centres, sig)
    if metric == "ip":
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        q /= np.linalg.norm(q, axis=1, keepdims=True)
    return Workload(f"tiny{d}", x.astype(np.float32), q.astype(np.float32), metric, 8, 64, 32, 5, seed)


def gen_grid(n=800, d=16, nq=20, seed=0):
    """Lossless-grid fixture: integer data in [0,255], every dimension holds
    both 0 and 255.  With P_l=0, P_h=100 the quantizer maps x -> x exactly."""
    r = _rng(seed, "grid", 0)
    x = r.integers(0, 256, size=(n, d)).astype(np.float32)
    x[0, :] = 0.0
    x[1, :] = 255.0
    q = _rng(seed, "grid", 1).integers(0, 256, size=(nq, d)).astype(np.float32)
    return Workload("grid", x, q, "l2", 8, 64, 32, 5, seed)


# ---------------------------------------------------------------------------------
# random numbers the method draws
# ---------------------------------------------------------------------------------

def density_sample(n: int, seed: int = 0, cfg: str = "C2", threshold: int = 10_000, cap: int = 5_000) -> np.ndarray:
    """Sorted int32 indices of the density sample (n > threshold -> min(cap, n) points, else all)."""
    if n <= threshold:
        return np.arange(n, dtype=np.int32)
    idx = _rng(seed, cfg, 2).choice(n, size=min(cap, n), replace=False)
    return np.sort(idx).astype(np.int32)


def level_draws(n: int, seed: int = 0, cfg: str = "C2", shard: int | None = None) -> np.ndarray:
    """U in (0, 1] per node, in insertion (id) order, for the HNSW level assignment (C5: one
    independent stream per shard)."""
    if shard is None:
        r = _rng(seed, cfg, 4)
    else:
        r = np.random.default_rng(np.random.SeedSequence([int(seed), CFG_IDS.get(cfg, 99), 4, int(shard)]))
    return (1.0 - r.random(n)).astype(np.float64)


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
