"""The cooperative kernel (warps_per_query = 4: one CTA of 4 warps per query, search.cu
coop_kernel) against the oracle through the C ABI, bit-exact like the one-warp kernel: visit
order, C and d^q, A and d^a, re-rank depth, ET flag, d^e, final ids and distances.  With no
visited set or the exact bitmap the per-query counters must equal the one-warp kernel's too
(the hash's re-evaluations depend on the order of inserts within a row, R15).

Covers every row shape the launcher dispatches on (LPR 1..32 via d = 7 .. 960, CAP 56 / 160),
both metrics, all visited modes, an ef whose W insert takes several move rounds, single queries,
and ef 8192 on a 960-d slice, where auto picks the cooperative kernel (W fills the SM)."""
import numpy as np
import pytest

import oracle
from tests._cases import case
from tests.test_gpu_configs import _parity, _upload

pytestmark = pytest.mark.gpu


def _counters(ix, q, p, vb, wpq):
    import torch
    import paper_2602_21600_b200 as aqr
    _, _, tr = aqr.search(ix, torch.from_numpy(np.ascontiguousarray(q)).cuda(), trace=True, exp_cap=4096,
                          visited_bits=vb, warps_per_query=wpq, **p)
    return tr["counters"].cpu().numpy()


@pytest.mark.parametrize("name", ["tiny7", "tiny33", "tiny100ip", "tiny960", "grid", "c1small", "c2slice", "c4slice"])
@pytest.mark.parametrize("vb", [-1, -2, 10])
@pytest.mark.parametrize("ef", [48, 400])
def test_coop_parity(name, vb, ef):
    c = case(name)
    ix = _upload(c)
    p = dict(k=c.w.k, **oracle.ef_mapping(ef, c.w.k))
    q = c.w.q[:16]
    _parity(c.ix, ix, q, p, vb, f"{name} coop vb{vb} ef{ef}", warps_per_query=4)
    if vb != 10:
        np.testing.assert_array_equal(_counters(ix, q, p, vb, 4)[:, :13], _counters(ix, q, p, vb, 1)[:, :13],
                                      err_msg=f"{name} coop counters")


@pytest.mark.parametrize("vb", [-1, -2])
def test_coop_large_ef_full_rerank(vb):
    """ef 2048 on the 60k C2 slice: the W insert moves > 256 entries (several rounds); full re-rank."""
    c = case("c2slice")
    ix = _upload(c)
    p = dict(k=c.w.k, **oracle.ef_mapping(2048, c.w.k))
    p["n_rerank"] = p["n_coarse"]
    _parity(c.ix, ix, c.w.q[:12], p, vb, f"c2slice coop ef2048 vb{vb}", warps_per_query=4)


def test_coop_single_query_and_auto():
    """nq = 1 (one CTA) with warps_per_query 4, and auto vs one warp: identical results."""
    import torch
    import paper_2602_21600_b200 as aqr
    c = case("c1small")
    ix = _upload(c)
    p = dict(k=c.w.k, **oracle.ef_mapping(96, c.w.k))
    _parity(c.ix, ix, c.w.q[:1], p, -1, "c1small coop nq1", warps_per_query=4)
    q = torch.from_numpy(np.ascontiguousarray(c.w.q[:3])).cuda()
    a = aqr.search(ix, q, warps_per_query=0, **p)
    b = aqr.search(ix, q, warps_per_query=1, **p)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a[0].cpu().numpy(), b[0].cpu().numpy())
    np.testing.assert_array_equal(a[1].cpu().numpy().view(np.uint32), b[1].cpu().numpy().view(np.uint32))


def test_coop_rejected_combinations():
    import torch
    import paper_2602_21600_b200 as aqr
    c = case("tiny33")
    ix = _upload(c)
    inl = _upload(c, layout="inline")
    q = torch.from_numpy(np.ascontiguousarray(c.w.q[:2])).cuda()
    p = dict(k=c.w.k, **oracle.ef_mapping(48, c.w.k))
    with pytest.raises(aqr.AqrError):
        aqr.search(ix, q, warps_per_query=4, traversal="fp32", **p)
    with pytest.raises(aqr.AqrError):
        aqr.search(inl, q, warps_per_query=4, **p)
    with pytest.raises(aqr.AqrError):
        aqr.search(ix, q, warps_per_query=2, **p)


def test_coop_auto_large_ef_wide_rows():
    """ef 8192 (the ABI maximum; W = 64 KB per query) on the 960-d C4 slice: the one-warp launch
    holds <= 4 queries per SM, so auto (0) runs the cooperative kernel; bit-exact with the oracle
    and identical to an explicit warps_per_query = 4."""
    import torch
    import paper_2602_21600_b200 as aqr
    c = case("c4slice")
    ix = _upload(c)
    p = dict(k=c.w.k, **oracle.ef_mapping(8192, c.w.k))
    _parity(c.ix, ix, c.w.q[:4], p, -2, "c4slice auto ef8192", warps_per_query=0)
    q = torch.from_numpy(np.ascontiguousarray(c.w.q[:4])).cuda()
    a = aqr.search(ix, q, warps_per_query=0, visited_bits=-2, **p)
    b = aqr.search(ix, q, warps_per_query=4, visited_bits=-2, **p)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a[0].cpu().numpy(), b[0].cpu().numpy())
    # the plan query reports the launch auto makes: 4 warps here, one warp at a small ef
    assert aqr.search_plan(ix, 4, aqr.make_params(c.w.k, **oracle.ef_mapping(8192, c.w.k))) == 4
    assert aqr.search_plan(ix, 4, aqr.make_params(c.w.k, **oracle.ef_mapping(64, c.w.k))) == 1
    assert aqr.search_plan(ix, 4, aqr.make_params(c.w.k, **oracle.ef_mapping(64, c.w.k), warps_per_query=4)) == 4
