"""GPU edge cases through the C ABI, each against the CPU oracle on the same seeded inputs:
empty and ragged query batches, indexes smaller than k (padding), a single-layer graph, exact
duplicate base vectors (ties broken by id), d = 1, the largest ef / k the ABI accepts,
and host-side argument errors."""
import numpy as np
import pytest

import oracle
import synth
from tests._cases import _mk

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _aqr():
    import paper_2602_21600_b200 as aqr
    return aqr


def _gpu_index(c, layout="gather"):
    torch = _torch()
    aqr = _aqr()
    x = torch.from_numpy(c.w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(c.sample).cuda(), p_max=5.0,
                              delta_override=c.delta_override)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(codes.cpu().numpy(), c.codes)
    return aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric, layout=layout)


def _compare(c, ix, q, p, exp_cap=4096):
    """visit order, C, final ids and final distances bit-exact (R24)."""
    torch = _torch()
    aqr = _aqr()
    o_ids, o_d, o_tr = oracle.search(c.ix, q, trace=True, exp_cap=exp_cap, **p)
    g_ids, g_d, g_tr = aqr.search(ix, torch.from_numpy(q).cuda(), trace=True, exp_cap=exp_cap, **p)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g_tr["exp_ids"].cpu().numpy(), o_tr["exp_ids"])
    np.testing.assert_array_equal(g_tr["coarse_ids"].cpu().numpy(), o_tr["coarse_ids"])
    np.testing.assert_array_equal(g_tr["coarse_dq"].cpu().numpy(), o_tr["coarse_dq"])
    np.testing.assert_array_equal(g_ids.cpu().numpy(), o_ids)
    g_d = g_d.cpu().numpy()
    fin = np.isfinite(o_d)
    np.testing.assert_array_equal(np.isfinite(g_d), fin)
    np.testing.assert_array_equal(g_d.view(np.uint32), o_d.view(np.uint32))
    return g_ids.cpu().numpy(), g_d


def test_empty_batch():
    torch = _torch()
    aqr = _aqr()
    c = _mk("e0", synth.gen_tiny(n=300, d=16, nq=4), M=6, efc=32)
    ix = _gpu_index(c)
    q = torch.empty((0, 16), dtype=torch.float32, device="cuda")
    ids, d = aqr.search(ix, q, k=5, ef=16, n_coarse=8, n_rerank=8)
    torch.cuda.synchronize()
    assert ids.shape == (0, 5) and d.shape == (0, 5)


@pytest.mark.parametrize("nq", [1, 3, 33, 131])
def test_ragged_batches(nq):
    c = _mk(f"rag{nq}", synth.gen_tiny(n=900, d=24, nq=nq, seed=nq), M=8, efc=48)
    ix = _gpu_index(c)
    _compare(c, ix, c.w.q, dict(k=7, ef=40, n_coarse=13, n_rerank=9))


def test_index_smaller_than_k_pads():
    # n = 12 < k = 16 (the density kNN needs n > 10): every query returns the 12 nodes, then
    # (-1, +inf)
    c = _mk("small", synth.gen_tiny(n=12, d=5, nq=5), M=4, efc=12)
    ix = _gpu_index(c)
    ids, d = _compare(c, ix, c.w.q, dict(k=16, ef=16, n_coarse=16, n_rerank=16, early_term=False))
    assert (ids[:, 12:] == -1).all() and np.isinf(d[:, 12:]).all()
    assert (np.sort(ids[:, :12], axis=1) == np.arange(12)).all()


def test_single_layer_graph():
    c = _mk("flat", synth.gen_tiny(n=30, d=9, nq=6), M=40, efc=40)
    assert c.graph.max_level == 0  # no upper layer: the descent is empty, layer 0 starts at the entry
    ix = _gpu_index(c)
    _compare(c, ix, c.w.q, dict(k=5, ef=16, n_coarse=8, n_rerank=8))


def test_duplicate_vectors_tie_by_id():
    w = synth.gen_tiny(n=400, d=12, nq=10)
    w.x[200:400] = w.x[0:200]  # every vector twice: exact d^q, d^a and d^e ties
    w.q[:5] = w.x[[3, 50, 120, 199, 0]]  # queries sitting on duplicated points
    c = _mk("dups", w, M=8, efc=48)
    ix = _gpu_index(c)
    ids, _ = _compare(c, ix, w.q, dict(k=6, ef=48, n_coarse=16, n_rerank=16, early_term=False))
    # each self-query returns the lower id of the pair first (ties by id)
    for qi, j in enumerate([3, 50, 120, 199, 0]):
        assert list(ids[qi, :2]) == [j, j + 200]


def test_one_dimension():
    c = _mk("d1", synth.gen_tiny(n=500, d=1, nq=12), M=4, efc=24)
    ix = _gpu_index(c)
    _compare(c, ix, c.w.q, dict(k=4, ef=24, n_coarse=8, n_rerank=8))


@pytest.mark.parametrize("layout", ["gather", "inline"])
def test_largest_ef_and_k(layout):
    # ef = 4096 over a 3000-node index: W holds the whole reachable set; k = 100 (C5's k) with
    # N_c = N_rerank = 100
    from tests._cases import case
    c = case("c1small")
    ix = _gpu_index(c, layout)
    _compare(c, ix, c.w.q[:8], dict(k=100, ef=4096, n_coarse=100, n_rerank=100))


def test_ef_8192():
    # the ABI maximum ef = 8192 (64 KB of W per query: one warp per CTA) on the 60k C2 slice,
    # where W really fills: the 13-step lower bound, the long W moves and a 2730-entry C
    from tests._cases import case
    c = case("c2slice")
    ix = _gpu_index(c)
    _compare(c, ix, c.w.q[:6], dict(k=10, ef=8192, n_coarse=2730, n_rerank=2730), exp_cap=16384)


def test_argument_errors():
    torch = _torch()
    aqr = _aqr()
    c = _mk("err", synth.gen_tiny(n=200, d=8, nq=2), M=4, efc=16)
    ix = _gpu_index(c)
    q = torch.from_numpy(c.w.q).cuda()
    with pytest.raises(aqr.AqrError, match="ef >= n_coarse"):
        aqr.search(ix, q, k=5, ef=8, n_coarse=10, n_rerank=5)
    with pytest.raises(aqr.AqrError, match="n_coarse >= k"):
        aqr.search(ix, q, k=12, ef=16, n_coarse=10, n_rerank=5)
    with pytest.raises(aqr.AqrError, match="ef > 8192"):
        aqr.search(ix, q, k=5, ef=9000, n_coarse=10, n_rerank=5)
    with pytest.raises(aqr.AqrError):
        aqr.search(ix, q.cpu(), k=5, ef=16, n_coarse=10, n_rerank=5)  # host tensor: no CPU path
