"""The exact global visited bitmap (visited_bits = -2; R15): one n-bit map per warp slot in the
caller's workspace.  Visit order, C, ids and distances must be exactly those of the default
(no visited set) and of the oracle, and the kernel's layer-0 evaluation count must then equal
the oracle's count of DISTINCT evaluations (its exact visited set) query by query."""
import numpy as np
import pytest

import oracle
from tests._cases import case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["tiny33", "tiny960", "c1small", "c2slice", "grid"])
@pytest.mark.parametrize("traversal", ["aqr", "fp32"])
def test_visited_bitmap_exact(name, traversal):
    import torch
    import paper_2602_21600_b200 as aqr
    c = case(name)
    x = torch.from_numpy(c.w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(c.sample).cuda(), p_max=5.0,
                              delta_override=c.delta_override)
    ix = aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric, layout="gather")
    k = c.w.k
    p = dict(k=k, **oracle.ef_mapping(96, k))
    q = torch.from_numpy(c.w.q).cuda()
    o_ids, o_d, o_tr = oracle.search(c.ix, c.w.q, trace=True, exp_cap=4096, traversal=traversal, **p)
    runs = {}
    for vb in (-1, -2):
        runs[vb] = aqr.search(ix, q, trace=True, exp_cap=4096, visited_bits=vb, traversal=traversal, **p)
    torch.cuda.synchronize()
    (i1, d1, t1), (i2, d2, t2) = runs[-1], runs[-2]
    np.testing.assert_array_equal(i2.cpu().numpy(), i1.cpu().numpy())
    np.testing.assert_array_equal(d2.cpu().numpy().view(np.uint32), d1.cpu().numpy().view(np.uint32))
    np.testing.assert_array_equal(t2["exp_ids"].cpu().numpy(), o_tr["exp_ids"])
    np.testing.assert_array_equal(t2["coarse_ids"].cpu().numpy(), o_tr["coarse_ids"])
    np.testing.assert_array_equal(t2["coarse_dq"].cpu().numpy(), o_tr["coarse_dq"])
    gc, oc = t2["counters"].cpu().numpy(), o_tr["counters"]
    np.testing.assert_array_equal(gc[:, 0], oc[:, 0])  # expansions
    np.testing.assert_array_equal(gc[:, 1], oc[:, 1])  # layer-0 neighbours seen
    np.testing.assert_array_equal(gc[:, 2], oc[:, 2])  # distinct evaluations, exactly
    # without the bitmap every neighbour is scored
    np.testing.assert_array_equal(t1["counters"].cpu().numpy()[:, 2], oc[:, 1])


def test_visited_bitmap_workspace_bound():
    """A workspace with only 8 bitmaps: the persistent grid shrinks to 8 warps and still serves
    all 2,000 queries with the default results."""
    import torch
    import paper_2602_21600_b200 as aqr
    c = case("c1small")
    x = torch.from_numpy(c.w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(c.sample).cuda(), p_max=5.0)
    ix = aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric, layout="gather")
    q = torch.from_numpy(np.tile(c.w.q, (50, 1))).cuda()  # 2,000 queries
    p = aqr.make_params(c.w.k, **oracle.ef_mapping(64, c.w.k), visited_bits=-2)
    s = aqr.Searcher(ix, len(q), p)
    words = (len(c.w.x) + 127) // 128 * 4
    s.ws = torch.zeros(256 + 8 * words * 4, dtype=torch.uint8, device="cuda")  # 8 bitmap slots
    ids, _ = s.run(q)
    ref, _ = aqr.search(ix, q, c.w.k, **oracle.ef_mapping(64, c.w.k))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ids.cpu().numpy(), ref.cpu().numpy())
