"""Pins of the oracle's FP32-HNSW baseline mode (the paper's comparison system "HNSW", P:207;
SURVEY 8(f) NEXT-2; R22): exact fp32 distances in the canonical order R(L), greedy
descent + flag-form beam on them, result = the first k of W."""
import numpy as np
import pytest

import oracle
import synth
from tests._cases import case


@pytest.mark.parametrize("d", [1, 7, 8, 9, 33, 100, 128, 960])
@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_fp_distance_within_fp64_bound(d, metric):
    rng = np.random.default_rng(d)
    for _ in range(20):
        q = rng.standard_normal(d).astype(np.float32)
        x = rng.standard_normal(d).astype(np.float32)
        got = oracle.dist_fp_RL(q, x, metric)
        if metric == "l2":
            ref = float(((q.astype(np.float64) - x) ** 2).sum())
            assert abs(got - ref) <= 1e-5 * ref
        else:
            dot = float((q.astype(np.float64) * x).sum())
            assert abs(got - (1.0 - dot)) <= 1e-5 * max(1.0, abs(dot))


def test_fp_distance_exact_on_integers():
    # integer coordinates with sums < 2^24: every fp32 partial is exact, so any summation
    # order gives the integer closed form
    rng = np.random.default_rng(1)
    for d in [3, 16, 128, 960]:
        q = rng.integers(0, 12, d).astype(np.float32)
        x = rng.integers(0, 12, d).astype(np.float32)
        assert oracle.dist_fp_RL(q, x) == float(((q.astype(np.int64) - x.astype(np.int64)) ** 2).sum())
        assert oracle.dist_fp_RL(q, x, "ip") == np.float32(1.0) - np.float32((q.astype(np.int64) * x.astype(np.int64)).sum())


@pytest.mark.parametrize("name", ["tiny33", "tiny100ip"])
def test_fp_search_exhaustive_is_bruteforce(name):
    """ef >= n reaches every node of the connected graph: the baseline returns the exact top-k."""
    c = case(name)
    n = len(c.w.x)
    k = 8
    ids, d = oracle.search(c.ix, c.w.q, k, ef=n, n_coarse=k, n_rerank=k, traversal="fp32")
    x64 = c.w.x.astype(np.float64)
    for i, qv in enumerate(c.w.q.astype(np.float64)):
        if c.w.metric == "l2":
            ex = ((x64 - qv) ** 2).sum(1)
        else:
            ex = 1.0 - x64 @ qv
        order = np.lexsort((np.arange(n), ex))
        gap = np.diff(np.sort(ex)[: k + 1])
        if np.all(gap > 1e-5 * np.abs(np.sort(ex)[1: k + 1]).max()):  # no near-ties in the top k+1
            np.testing.assert_array_equal(ids[i], order[:k])
        np.testing.assert_allclose(d[i], ex[ids[i]], rtol=1e-5, atol=1e-6)


def test_fp_equals_aqr_on_lossless_grid():
    """on the lossless grid the codes ARE the data and fp32 sums of integers are
    exact, so the quantized traversal and the FP32 baseline expand the same nodes in the same
    order and return the same C."""
    c = case("grid")
    p = dict(k=5, ef=40, n_coarse=13, n_rerank=13, early_term=False)
    _, _, ta = oracle.search(c.ix, c.w.q, trace=True, **p)
    _, _, tf = oracle.search(c.ix, c.w.q, trace=True, traversal="fp32", **p)
    np.testing.assert_array_equal(ta["exp_ids"], tf["exp_ids"])
    np.testing.assert_array_equal(ta["coarse_ids"], tf["coarse_ids"])
    np.testing.assert_array_equal(ta["coarse_dq"].astype(np.float32), tf["coarse_dq"].view(np.float32))
