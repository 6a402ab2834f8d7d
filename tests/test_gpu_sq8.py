"""GPU parity of the plain SQ8 HNSW baseline (R23): delta = 0 codes
(aqr_encode with delta_override = 0), the graph built on them, traversal on the codes with no
early termination and N_rerank = N_c.  Codes, visit order, C and d^q bit-exact; Stages 2-3, the
final ids and distances bit-exact too (canonical fp32 order R(32) on both sides, R24)."""
import numpy as np
import pytest

import oracle
from tests._cases import case

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
    # Stages 2-3 sum in the canonical order R(32) on both sides (R24): bit-exact
    from tests.test_gpu_parity import assert_stage23_exact
    assert_stage23_exact(o_ids, o_d, o_tr, g_ids, g_d, g_tr, f"{name} sq8")
