"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (default
layout, warps per block and visited setting, the ef bench.py reports for C2): the oracle
trains its own quantizer and encodes every base vector (compared byte for byte with
aqr_encode), then searches a sample of queries one by one on the same graph; the GPU's visit
order, C (ids + integer d^q) and final ids must be bit-exact, final distances within 1e-5.

C1 (configs[0], 10k x 128): all 100 queries at ef = 64 (BJ).
C2 (configs[1], 1M x 128, the bench workload): 24 sampled queries at ef = 784 (the smallest
ef with recall@10 >= 0.98 in profiles/r01) and at ef = 64."""
import numpy as np
import pytest

import oracle
import synth
from paper_2602_21600_b200 import graph as G

pytestmark = pytest.mark.gpu

P_MAX = {"C1": 5.0, "C2": 0.2}  # bench.py P_MAX (R4)


def _build(cfg):
    import torch
    import paper_2602_21600_b200 as aqr
    w = synth.gen_config(cfg)
    sample = synth.density_sample(len(w.x), seed=w.seed, cfg=cfg)
    x = torch.from_numpy(w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(sample).cuda(), p_max=P_MAX[cfg], want_rho=True)
    torch.cuda.synchronize()
    oq = oracle.train(w.x, sample, p_max=P_MAX[cfg])
    oc = oracle.encode(w.x, oq)
    np.testing.assert_array_equal(codes.cpu().numpy(), oc)  # every code of the full base set
    assert quant.delta == oq.delta
    rho = oracle.density(w.x, sample)
    eta = G.eta_of(G.density_weights(w.x[sample], rho))
    M, efc = G.adapt_params(w.M0, w.efc0, oq.delta, eta)
    g = G.build_hnsw(oc, M, efc, synth.level_draws(len(w.x), seed=w.seed, cfg=cfg), 0, flags=1)
    ix = aqr.upload_index(codes, x, quant, g, metric=w.metric)
    return w, ix, oracle.Index(w.x, oc, oq, g, w.metric)


def _check(w, ix, oix, qidx, ef):
    import torch
    import paper_2602_21600_b200 as aqr
    m = aqr.ef_mapping(ef, w.k)
    q = np.ascontiguousarray(w.q[qidx])
    o_ids, o_d, o_tr = oracle.search(oix, q, w.k, trace=True, exp_cap=4096, **m)
    g_ids, g_d, g_tr = aqr.search(ix, torch.from_numpy(q).cuda(), w.k, trace=True, exp_cap=4096, **m)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g_tr["exp_ids"].cpu().numpy(), o_tr["exp_ids"])
    np.testing.assert_array_equal(g_tr["coarse_ids"].cpu().numpy(), o_tr["coarse_ids"])
    np.testing.assert_array_equal(g_tr["coarse_dq"].cpu().numpy(), o_tr["coarse_dq"])
    np.testing.assert_array_equal(g_ids.cpu().numpy(), o_ids)
    np.testing.assert_allclose(g_d.cpu().numpy(), o_d, rtol=1e-5)


def test_c1_full():
    w, ix, oix = _build("C1")
    _check(w, ix, oix, np.arange(len(w.q)), 64)


def test_c2_full_sampled():
    w, ix, oix = _build("C2")
    qidx = np.random.default_rng(11).choice(len(w.q), 24, replace=False)
    _check(w, ix, oix, qidx, 784)
    _check(w, ix, oix, qidx, 64)
