"""Per-query latency stamps (aqr_debug.t_ns, %globaltimer; Fig. 4 / P:266 via tools/latency.py):
every query gets start < end, the stamps do not change the results, and a query's service time
is bounded by the launch's own duration."""
import numpy as np
import pytest

import oracle
from tests._cases import case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["tiny33", "c1small"])
def test_timing_stamps(name):
    import torch
    import paper_2602_21600_b200 as aqr
    c = case(name)
    x = torch.from_numpy(c.w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(c.sample).cuda(), p_max=5.0,
                              delta_override=c.delta_override)
    ix = aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric)
    q = torch.from_numpy(c.w.q).cuda()
    s = aqr.Searcher(ix, len(q), aqr.make_params(c.w.k, **oracle.ef_mapping(64, c.w.k)))
    ids0 = s.run(q)[0].clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ids1 = s.run(q, timing=True)[0].clone()
    e1.record()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ids0.cpu().numpy(), ids1.cpu().numpy())
    t = s.t_ns[: len(q)].cpu().numpy()
    assert (t[:, 0] > 0).all() and (t[:, 1] > t[:, 0]).all()
    span_ms = (t[:, 1].max() - t[:, 0].min()) / 1e6
    assert span_ms <= e0.elapsed_time(e1) + 0.05
    assert s.totals.sum().item() == 0  # timing alone collects no counters
