"""Pins of the plain SQ8 HNSW baseline (R23; the paper's "Scalar Quantization" comparison, P:207;
SURVEY 8(f) NEXT-2): delta = 0 codes (full-range min/max, pinned in test_oracle_pins), traversal on
those codes, no early termination and every C entry re-ranked exactly.  With N_rerank = N_c the
result is fixed by a plain definition: the k entries of C nearest to q in exact distance, which
numpy computes here in fp64 from the oracle's own C list."""
import numpy as np
import pytest

import oracle
from tests._cases import case


def _exact(x, q, metric):
    x = x.astype(np.float64)
    q = q.astype(np.float64)
    if metric == "l2":
        return ((x - q) ** 2).sum(-1)
    return 1.0 - x @ q


@pytest.mark.parametrize("name", ["tiny33_sq8", "tiny100ip_sq8", "c1small_sq8"])
@pytest.mark.parametrize("ef", [16, 96])
def test_sq8_full_rerank_is_exact_topk_of_C(name, ef):
    c = case(name)
    assert c.quant.delta == 0.0
    np.testing.assert_array_equal(c.quant.min_f, c.w.x.min(0))
    np.testing.assert_array_equal(c.quant.max_f, c.w.x.max(0))
    k = c.w.k
    m = oracle.ef_mapping(ef, k)
    m["n_rerank"] = m["n_coarse"]
    ids, d, tr = oracle.search(c.ix, c.w.q, k, trace=True, early_term=False, **m)
    for i in range(len(c.w.q)):
        cids = tr["coarse_ids"][i]
        cids = cids[cids >= 0]
        ex = _exact(c.w.x[cids], c.w.q[i], c.w.metric)
        order = np.lexsort((cids, ex))[:k]
        want_d = ex[order]
        got = ids[i][ids[i] >= 0]
        assert len(got) == min(k, len(cids))
        np.testing.assert_allclose(d[i][: len(got)], want_d, rtol=1e-5, atol=1e-6)
        # ids agree except where fp32 rounding can swap a near-tie
        srt = np.sort(ex)
        tie = np.any(np.isclose(srt[1:], srt[:-1], rtol=2e-5, atol=1e-7)) if len(srt) > 1 else False
        if not tie:
            np.testing.assert_array_equal(got, cids[order])
        # no early termination: every C entry was re-ranked
        assert tr["counters"][i, 7] == len(cids)
