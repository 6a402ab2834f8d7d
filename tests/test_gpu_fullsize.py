"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (default
layout, warps per block and visited setting, the ef bench.py reports for C2): the oracle
trains its own quantizer and encodes every base vector (compared byte for byte with
aqr_encode), then searches a sample of queries one by one on the same graph; the GPU's visit
order, C (ids + integer d^q), Stages 2-3 (A, d^a, depth, ET flag, d^e) and the final ids and
distances must be bit-exact (canonical fp32 order R(32), R24).

C1 (configs[0], 10k x 128): all 100 queries at ef = 64 (BJ).
C2 (configs[1], 1M x 128, the bench workload): 24 sampled queries at ef = 784 (the smallest
ef with recall@10 >= 0.98 in profiles/r01) and at ef = 64."""
import os

import numpy as np
import pytest

import oracle
import synth
from paper_2602_21600_b200 import graph as G
from tests.test_gpu_parity import assert_stage23_exact

pytestmark = pytest.mark.gpu

P_MAX = {"C1": 0.2, "C2": 0.2, "C4": 0.2}  # bench.py P_MAX (R4)


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


def _check(w, ix, oix, qidx, ef, full=False, visited_bits=0):
    import torch
    import paper_2602_21600_b200 as aqr
    m = aqr.ef_mapping(ef, w.k)
    if full:
        m["n_rerank"] = m["n_coarse"]
    q = np.ascontiguousarray(w.q[qidx])
    o_ids, o_d, o_tr = oracle.search(oix, q, w.k, trace=True, exp_cap=4096, **m)
    g_ids, g_d, g_tr = aqr.search(ix, torch.from_numpy(q).cuda(), w.k, trace=True, exp_cap=4096,
                                  visited_bits=visited_bits, **m)
    torch.cuda.synchronize()
    g_tr = {kk: v.cpu().numpy() for kk, v in g_tr.items()}
    np.testing.assert_array_equal(g_tr["exp_ids"], o_tr["exp_ids"])
    np.testing.assert_array_equal(g_tr["coarse_ids"], o_tr["coarse_ids"])
    np.testing.assert_array_equal(g_tr["coarse_dq"], o_tr["coarse_dq"])
    assert_stage23_exact(o_ids, o_d, o_tr, g_ids.cpu().numpy(), g_d.cpu().numpy(), g_tr, f"{w.name} ef{ef}")


def test_c1_full():
    w, ix, oix = _build("C1")
    _check(w, ix, oix, np.arange(len(w.q)), 64)


def test_c2_full_sampled():
    w, ix, oix = _build("C2")
    qidx = np.random.default_rng(11).choice(len(w.q), 24, replace=False)
    _check(w, ix, oix, qidx, 784)
    _check(w, ix, oix, qidx, 64)


@pytest.mark.skipif(not os.environ.get("AQR_FULL_C4"), reason="~10 min (1M x 960 host graph build); AQR_FULL_C4=1")
def test_c4_full_sampled():
    """BASELINE configs[3] at full size (1M x 960, M adapted to 70): the bench's point, ef 1536 with a
    full re-rank and the exact global bitmap (visited_bits -2), 12 sampled queries.  Run on demand
    (profiles/r02/gputest_c4_full.log): the host graph build alone takes ~7 min on the box."""
    w, ix, oix = _build("C4")
    qidx = np.random.default_rng(17).choice(len(w.q), 12, replace=False)
    _check(w, ix, oix, qidx, 1536, full=True, visited_bits=-2)
