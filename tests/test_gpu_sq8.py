"""GPU parity of the plain SQ8 HNSW baseline (R23): delta = 0 codes
(aqr_encode with delta_override = 0), the graph built on them, traversal on the codes with no
early termination and N_rerank = N_c.  Codes, visit order, C and d^q bit-exact; final ids exact
unless an fp32 near-tie explains the difference; distances within 1e-5 relative."""
import numpy as np
import pytest

import oracle
from tests._cases import case, near

pytestmark = pytest.mark.gpu

CASES = ["tiny33_sq8", "tiny100ip_sq8", "tiny960_sq8", "c1small_sq8", "c2slice_sq8"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("ef", [16, 96])
def test_sq8_parity(name, ef):
    import torch
    import paper_2602_21600_b200 as aqr
    c = case(name)
    x = torch.from_numpy(c.w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(c.sample).cuda(), p_max=5.0, delta_override=0.0)
    torch.cuda.synchronize()
    assert quant.delta == 0.0
    np.testing.assert_array_equal(codes.cpu().numpy(), c.codes)
    ix = aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric)
    k = c.w.k
    m = oracle.ef_mapping(ef, k)
    m["n_rerank"] = m["n_coarse"]
    o_ids, o_d, o_tr = oracle.search(c.ix, c.w.q, k, trace=True, exp_cap=4096, early_term=False, **m)
    g_ids, g_d, g_tr = aqr.search(ix, torch.from_numpy(c.w.q).cuda(), k, trace=True, exp_cap=4096,
                                  early_term=False, **m)
    torch.cuda.synchronize()
    g_ids, g_d = g_ids.cpu().numpy(), g_d.cpu().numpy()
    g_tr = {kk: v.cpu().numpy() for kk, v in g_tr.items()}
    np.testing.assert_array_equal(g_tr["exp_ids"], o_tr["exp_ids"])
    np.testing.assert_array_equal(g_tr["coarse_ids"], o_tr["coarse_ids"])
    np.testing.assert_array_equal(g_tr["coarse_dq"], o_tr["coarse_dq"])
    np.testing.assert_array_equal(g_tr["counters"][:, 7], o_tr["counters"][:, 7])  # every C entry re-ranked
    n_bad = 0
    for i in range(len(c.w.q)):
        if np.array_equal(o_ids[i], g_ids[i]):
            fin = np.isfinite(o_d[i])
            assert np.all(near(o_d[i][fin], g_d[i][fin], metric=c.w.metric)), (i, o_d[i], g_d[i])
            continue
        n_bad += 1
        ex = np.sort(o_tr["exact_d"][i][np.isfinite(o_tr["exact_d"][i])])
        assert np.any(near(ex[1:], ex[:-1], 2e-5, c.w.metric)), (i, o_ids[i], g_ids[i])
    assert n_bad <= max(1, len(c.w.q) // 20)
