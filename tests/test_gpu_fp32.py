"""GPU parity of the FP32-HNSW baseline traversal (AQR_TRAVERSAL_FP32):
the same graph searched on exact fp32 distances.  Both sides use the canonical summation
order R(L) (R22), so visit order, C, ids AND distances are bit-exact."""
import numpy as np
import pytest

import oracle
from tests._cases import case

pytestmark = pytest.mark.gpu

CASES = ["tiny7", "tiny33", "tiny100ip", "tiny960", "grid", "c1small", "c2slice"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("ef", [16, 96])
def test_fp32_traversal_bit_exact(name, ef):
    import torch
    import paper_2602_21600_b200 as aqr
    c = case(name)
    x = torch.from_numpy(c.w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(c.sample).cuda(), p_max=5.0,
                              delta_override=c.delta_override)
    ix = aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric)
    k = c.w.k
    p = dict(k=k, ef=ef, n_coarse=min(ef, max(k, 12)), n_rerank=k)
    o_ids, o_d, o_tr = oracle.search(c.ix, c.w.q, trace=True, exp_cap=4096, traversal="fp32", **p)
    g_ids, g_d, g_tr = aqr.search(ix, torch.from_numpy(c.w.q).cuda(), trace=True, exp_cap=4096,
                                  traversal="fp32", **p)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g_tr["exp_ids"].cpu().numpy(), o_tr["exp_ids"])
    np.testing.assert_array_equal(g_tr["coarse_ids"].cpu().numpy(), o_tr["coarse_ids"])
    np.testing.assert_array_equal(g_tr["coarse_dq"].cpu().numpy(), o_tr["coarse_dq"])
    np.testing.assert_array_equal(g_ids.cpu().numpy(), o_ids)
    np.testing.assert_array_equal(g_d.cpu().numpy().view(np.uint32), o_d.view(np.uint32))
    np.testing.assert_array_equal(g_tr["counters"].cpu().numpy()[:, 0], o_tr["counters"][:, 0])
