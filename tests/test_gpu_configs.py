"""GPU parity of the kernel configurations the other files do not reach, each
bit-exact against the oracle through the C ABI (visit order, C and d^q, A and d^a, re-rank depth,
ET flag, d^e, final ids and distances):

* c4slice: 960-d rows (LPR 32: one row per warp step, the TMA-staged wide-row gather when the
  launcher picks it) with C4's adapted degree class (M = 35: 70-entry layer-0 rows, CAP 160), at
  the bench's settings for C4 -- full re-rank, no visited set and the exact global bitmap (-2);
* the shared-memory visited hash at 2^12 / 2^13 slots (the sizes bench.py tries on C1) on c1small
  and c2slice, where the kernel may also forget ids (R15): results must not change;
* the full-size C3 base (1.18M x 100, inner product) on sampled queries at the bench's ef 1536
  with a full re-rank, in the default launch configuration.
"""
import numpy as np
import pytest

import oracle
from tests._cases import case
from tests.test_gpu_parity import assert_stage23_exact

pytestmark = pytest.mark.gpu


def _upload(c, layout="gather"):
    import torch
    import paper_2602_21600_b200 as aqr
    x = torch.from_numpy(c.w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(c.sample).cuda(), p_max=5.0,
                              delta_override=c.delta_override)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(codes.cpu().numpy(), c.codes)
    return aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric, layout=layout)


def _parity(oix, ix, q, p, visited_bits=-1, ctx="", **gkw):
    import torch
    import paper_2602_21600_b200 as aqr
    o_ids, o_d, o_tr = oracle.search(oix, q, trace=True, exp_cap=4096, **p)
    g_ids, g_d, g_tr = aqr.search(ix, torch.from_numpy(np.ascontiguousarray(q)).cuda(), trace=True, exp_cap=4096,
                                  visited_bits=visited_bits, **p, **gkw)
    torch.cuda.synchronize()
    g_tr = {k: v.cpu().numpy() for k, v in g_tr.items()}
    np.testing.assert_array_equal(g_tr["exp_ids"], o_tr["exp_ids"], err_msg=f"{ctx} visit order")
    np.testing.assert_array_equal(g_tr["coarse_ids"], o_tr["coarse_ids"], err_msg=f"{ctx} C")
    np.testing.assert_array_equal(g_tr["coarse_dq"], o_tr["coarse_dq"], err_msg=f"{ctx} C d^q")
    np.testing.assert_array_equal(g_tr["counters"][:, 3:6], o_tr["counters"][:, 3:6], err_msg=f"{ctx} upper")
    assert_stage23_exact(o_ids, o_d, o_tr, g_ids.cpu().numpy(), g_d.cpu().numpy(), g_tr, ctx)
    return g_tr, o_tr


@pytest.mark.parametrize("ef", [96, 256])
@pytest.mark.parametrize("vb", [-1, -2, 8, 12])
def test_c4slice_wide_rows_cap160(ef, vb):
    """The wide-row (TMA-staged) kernel with every visited mode; vb 8 / 12 put the shared-memory
    hash beside the stage buffer (they once shared one region: staged rows overwrote the table)."""
    c = case("c4slice")
    assert c.graph.M == 35 and c.w.x.shape[1] == 960
    ix = _upload(c)
    p = dict(k=c.w.k, **oracle.ef_mapping(ef, c.w.k))
    p["n_rerank"] = p["n_coarse"]  # the bench's C4 mapping ("full", R20)
    g_tr, o_tr = _parity(c.ix, ix, c.w.q, p, vb, f"c4slice ef{ef} vb{vb}")
    if vb == -2:  # the exact bitmap: the kernel scores each node once, as the oracle does
        np.testing.assert_array_equal(g_tr["counters"][:, 2], o_tr["counters"][:, 2])


@pytest.mark.parametrize("name", ["c1small", "c2slice"])
@pytest.mark.parametrize("vb", [6, 10, 12, 13])
def test_shared_memory_visited_hash(name, vb):
    """The direct-mapped table (16-bit tags of a bijective hash, R15) at sizes from thrashing (2^6
    slots: every slot rewritten many times per query) to roomy: results and visit order exact."""
    c = case(name)
    ix = _upload(c)
    p = dict(k=c.w.k, **oracle.ef_mapping(96, c.w.k))
    g_tr, o_tr = _parity(c.ix, ix, c.w.q, p, vb, f"{name} hash 2^{vb}")
    # the hash never skips a node the oracle scores (no false positives): it scores at least the
    # distinct nodes, at most every neighbour
    ev, distinct, seen = g_tr["counters"][:, 2], o_tr["counters"][:, 2], o_tr["counters"][:, 1]
    assert np.all(ev >= distinct) and np.all(ev <= seen)


def test_c3_full_size_sampled():
    """BASELINE configs[2] at full size (1.18M x 100, IP), 16 sampled queries at the bench's point:
    ef 1536, N_c 512, full re-rank (profiles/r01 bench_c3)."""
    import torch
    import synth
    import paper_2602_21600_b200 as aqr
    from paper_2602_21600_b200 import graph as G
    w = synth.gen_config("C3")
    sample = synth.density_sample(len(w.x), seed=w.seed, cfg="C3")
    x = torch.from_numpy(w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(sample).cuda(), p_max=5.0)
    torch.cuda.synchronize()
    oq = oracle.train(w.x, sample, p_max=5.0)
    oc = oracle.encode(w.x, oq)
    np.testing.assert_array_equal(codes.cpu().numpy(), oc)
    rho = oracle.density(w.x, sample)
    M, efc = G.adapt_params(w.M0, w.efc0, oq.delta, G.eta_of(G.density_weights(w.x[sample], rho)))
    g = G.build_hnsw(oc, M, efc, synth.level_draws(len(w.x), seed=w.seed, cfg="C3"), 0, flags=1)
    ix = aqr.upload_index(codes, x, quant, g, metric="ip")
    oix = oracle.Index(w.x, oc, oq, g, "ip")
    qidx = np.random.default_rng(13).choice(len(w.q), 16, replace=False)
    p = dict(k=w.k, **oracle.ef_mapping(1536, w.k))
    p["n_rerank"] = p["n_coarse"]
    _parity(oix, ix, w.q[qidx], p, -1, "C3 full ef1536")


@pytest.mark.parametrize("vb", [-1, 12, -2])
def test_fp32_traversal_on_inline_index(vb):
    """The FP32-HNSW baseline (R22) runs the GATHER kernel even on an INLINE index; with the visited
    hash its shared memory must hold the hash, not the INLINE block (found by tools/sanitize_run.py:
    an illegal address before the fix).  Bit-exact with the oracle's fp32 mode."""
    import torch
    import paper_2602_21600_b200 as aqr
    c = case("tiny33")
    ix = _upload(c, layout="inline")
    p = dict(k=c.w.k, **oracle.ef_mapping(48, c.w.k))
    o_ids, o_d, o_tr = oracle.search(c.ix, c.w.q, trace=True, traversal="fp32", **p)
    g_ids, g_d, g_tr = aqr.search(ix, torch.from_numpy(c.w.q).cuda(), trace=True, traversal="fp32", visited_bits=vb, **p)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g_tr["exp_ids"].cpu().numpy(), o_tr["exp_ids"])
    np.testing.assert_array_equal(g_ids.cpu().numpy(), o_ids)
    np.testing.assert_array_equal(g_d.cpu().numpy().view(np.uint32), o_d.view(np.uint32))
