"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): quantized codes, int32 d^q, visit order and returned ids
bit-exact (ties by id); fp32 re-rank distances within 1e-5 relative, ids differing only
inside such near-ties.
"""
import numpy as np
import pytest

import oracle
from tests._cases import case, near

pytestmark = pytest.mark.gpu

CASES = ["tiny7", "tiny33", "tiny100ip", "tiny960", "grid", "c1small", "c2slice"]


def _torch():
    import torch
    return torch


def _aqr():
    import paper_2602_21600_b200 as aqr
    return aqr


@pytest.fixture(scope="module")
def gpu_index():
    cache = {}

    def get(name):
        if name not in cache:
            torch = _torch()
            aqr = _aqr()
            c = case(name)
            x = torch.from_numpy(c.w.x).cuda()
            sample = torch.from_numpy(c.sample).cuda()
            codes, quant = aqr.encode(x, sample_idx=sample, p_max=5.0, delta_override=c.delta_override)
            torch.cuda.synchronize()
            ix = aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric, layout="gather")
            ixi = aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric, layout="inline")
            assert ix.layout == "gather" and ixi.layout == "inline"
            cache[name] = (c, codes, quant, ix, ixi)
        return cache[name]

    return get


@pytest.mark.parametrize("name", CASES)
def test_encode_bit_exact(gpu_index, name):
    c, codes, quant, _, _ = gpu_index(name)
    assert quant.delta == c.quant.delta
    np.testing.assert_array_equal(quant.min_j.cpu().numpy().view(np.uint32), c.quant.min_f.view(np.uint32))
    np.testing.assert_array_equal(quant.max_j.cpu().numpy().view(np.uint32), c.quant.max_f.view(np.uint32))
    np.testing.assert_array_equal(quant.scale_j.cpu().numpy().view(np.uint32), c.quant.scale_f.view(np.uint32))
    np.testing.assert_array_equal(codes.cpu().numpy(), c.codes)


def _params(c, ef):
    k = c.w.k
    m = oracle.ef_mapping(ef, k)
    return dict(k=k, **m)


def _explained(o_ad, k, depth_or, p, o_fd, g_fd, metric):
    """Is a final-list difference explained by an fp32 near-tie (1e-5 rel) at a decision point?"""
    n = len(o_ad)
    cuts = [depth_or, k]
    for cpos in cuts:
        if 0 < cpos < n and near(o_ad[cpos - 1], o_ad[cpos], 2e-5, metric):
            return True
    if n > k:  # early-termination test near its threshold
        ak, ak1 = float(o_ad[k - 1]), float(o_ad[k])
        gap = (ak1 - ak) / (ak + 1e-6)
        ratio = ak1 / (ak + 1e-6)
        if abs(gap - p["tau_gap"]) <= 1e-4 * max(1.0, abs(gap)) or abs(ratio - p["tau_ratio"]) <= 1e-4 * ratio:
            return True
    fd = np.concatenate([o_fd, g_fd])
    fd = np.sort(fd[np.isfinite(fd)])
    return bool(np.any(near(fd[1:], fd[:-1], 2e-5, metric)))


@pytest.mark.parametrize("layout", ["gather", "inline"])
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("ef", [16, 48, 96])
def test_search_parity(gpu_index, name, ef, layout):
    torch = _torch()
    aqr = _aqr()
    c, codes, quant, ixg, ixi = gpu_index(name)
    ix = ixg if layout == "gather" else ixi
    p = _params(c, ef)
    p.update(tau_gap=0.010, tau_ratio=1.008, early_term=True)
    q = c.w.q
    o_ids, o_d, o_tr = oracle.search(c.ix, q, trace=True, exp_cap=4096, **p)
    g_ids, g_d, g_tr = aqr.search(ix, torch.from_numpy(q).cuda(), trace=True, exp_cap=4096, **p)
    torch.cuda.synchronize()
    g_ids, g_d = g_ids.cpu().numpy(), g_d.cpu().numpy()
    g_tr = {k: v.cpu().numpy() for k, v in g_tr.items()}
    oc = o_tr["counters"]
    gc = g_tr["counters"]
    # Stage 1: visit order, |W| prefix C and its integer distances are bit-exact
    nexp = oc[:, 0]
    np.testing.assert_array_equal(gc[:, 0], nexp, err_msg="expansion counts")
    np.testing.assert_array_equal(g_tr["exp_ids"], o_tr["exp_ids"], err_msg="visit order")
    np.testing.assert_array_equal(g_tr["coarse_ids"], o_tr["coarse_ids"], err_msg="C ids")
    np.testing.assert_array_equal(g_tr["coarse_dq"], o_tr["coarse_dq"], err_msg="C d^q")
    # upper-layer greedy path is identical too
    np.testing.assert_array_equal(gc[:, 3], oc[:, 3])
    # Stage 2: A is a permutation of C; d^a within 1e-5 relative per id
    n_bad = 0
    for i in range(len(q)):
        nc = int(oc[i, 6])
        o_map = dict(zip(o_tr["asym_ids"][i, :nc], o_tr["asym_d"][i, :nc]))
        g_map = dict(zip(g_tr["asym_ids"][i, :nc], g_tr["asym_d"][i, :nc]))
        assert set(o_map) == set(g_map)
        for kk in o_map:
            assert near(o_map[kk], g_map[kk], metric=c.w.metric), (i, kk, o_map[kk], g_map[kk])
        # final ids exact unless explained by a near-tie
        if not np.array_equal(o_ids[i], g_ids[i]):
            n_bad += 1
            assert _explained(o_tr["asym_d"][i, :nc], p["k"], int(oc[i, 7]), p, o_d[i], g_d[i], c.w.metric), (i, o_ids[i], g_ids[i])
        else:
            fin = np.isfinite(o_d[i])
            assert np.all(near(o_d[i][fin], g_d[i][fin], metric=c.w.metric)), (i, o_d[i], g_d[i])
    assert n_bad <= max(1, len(q) // 20)


@pytest.mark.parametrize("name", ["tiny7", "c1small"])
def test_rerank_split_equals_fused(gpu_index, name):
    torch = _torch()
    aqr = _aqr()
    c, codes, quant, ix, _ = gpu_index(name)
    p = _params(c, 48)
    qd = torch.from_numpy(c.w.q).cuda()
    ids, d, tr = aqr.search(ix, qd, trace=True, **p)
    ids2, d2 = aqr.rerank(ix, qd, tr["coarse_ids"], p["k"], p["n_rerank"])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ids.cpu().numpy(), ids2.cpu().numpy())
    np.testing.assert_array_equal(d.cpu().numpy().view(np.uint32), d2.cpu().numpy().view(np.uint32))
    # and the oracle's standalone rerank on the same C lists agrees
    o_ids, o_d = oracle.rerank(c.ix, c.w.q, tr["coarse_ids"].cpu().numpy(), p["k"], p["n_rerank"])
    assert (o_ids == ids.cpu().numpy()).mean() > 0.97


def test_merge_topk_matches_oracle():
    torch = _torch()
    aqr = _aqr()
    rng = np.random.default_rng(3)
    S, nq, k = 8, 50, 20
    d = rng.integers(0, 40, size=(S, nq, k)).astype(np.float32) / 4  # many exact ties
    ids = np.stack([rng.permutation(10_000)[: nq * k].reshape(nq, k) + s * 10_000 for s in range(S)]).astype(np.int32)
    order = np.lexsort((ids, d), axis=-1)
    d = np.take_along_axis(d, order, -1)
    ids = np.take_along_axis(ids, order, -1)
    ids[0, 0, -3:] = -1
    d[0, 0, -3:] = np.inf
    od, oi = oracle.merge_topk(d, ids, k)
    gd, gi = aqr.merge_topk(torch.from_numpy(d).cuda(), torch.from_numpy(ids).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(gi.cpu().numpy(), oi)
    np.testing.assert_array_equal(gd.cpu().numpy(), od)


def test_lossless_grid_equals_bruteforce(gpu_index):
    """lossless quantizer + exhaustive settings -> brute-force exact top-k."""
    torch = _torch()
    aqr = _aqr()
    c, codes, quant, ix, _ = gpu_index("grid")
    n = len(c.w.x)
    k = 5
    ids, d = aqr.search(ix, torch.from_numpy(c.w.q).cuda(), k=k, ef=n, n_coarse=n, n_rerank=n, early_term=False)
    bf_ids, bf_d = oracle.bruteforce(c.w.x, c.w.q, k)
    np.testing.assert_array_equal(ids.cpu().numpy(), bf_ids)
