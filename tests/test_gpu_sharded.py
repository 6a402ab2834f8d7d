"""C5-style sharded search on one GPU: each shard is a complete AQR index
(its own quantizer and graph, ids offset by the shard's first row); the per-shard top-k lists
are merged by aqr_merge_topk.  The oracle searches the same shards and merges with its own
merge; ids must be bit-exact (ties by global id), distances within 1e-5."""
import numpy as np
import pytest

import oracle
import synth
from paper_2602_21600_b200 import graph as G
from paper_2602_21600_b200 import parallel as P

pytestmark = pytest.mark.gpu

S, N_SHARD, NQ, K = 4, 3000, 40, 100


def test_sharded_merge_matches_oracle():
    import torch
    import paper_2602_21600_b200 as aqr
    q = synth.gen_c5_queries(NQ)
    m = aqr.ef_mapping(128, K)
    g_lists, o_lists = [], []
    for s in range(S):
        x = synth.gen_c5_shard(s, N_SHARD)
        samp = synth.density_sample(N_SHARD, cfg="C5")
        oq = oracle.train(x, samp, p_max=5.0)
        oc = oracle.encode(x, oq)
        g = G.build_hnsw(oc, 16, 64, synth.level_draws(N_SHARD, cfg="C5", shard=s), 4, flags=1)
        base = P.shard_rows(S * N_SHARD, S, s)[0]
        xt = torch.from_numpy(x).cuda()
        codes, quant = aqr.encode(xt, sample_idx=torch.from_numpy(samp).cuda(), p_max=5.0)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(codes.cpu().numpy(), oc)
        ix = aqr.upload_index(codes, xt, quant, g, metric="l2", id_base=base)
        gi, gd = aqr.search(ix, torch.from_numpy(q).cuda(), K, **m)
        g_lists.append((gd, gi))
        oi, od = oracle.search(oracle.Index(x, oc, oq, g, "l2"), q, K, **m)
        oi = np.where(oi >= 0, oi + base, -1).astype(np.int32)
        o_lists.append((od, oi))
    gd, gi = aqr.merge_topk(torch.stack([d for d, _ in g_lists]), torch.stack([i for _, i in g_lists]))
    torch.cuda.synchronize()
    od, oi = oracle.merge_topk(np.stack([d for d, _ in o_lists]), np.stack([i for _, i in o_lists]), K)
    np.testing.assert_array_equal(gi.cpu().numpy(), oi)
    np.testing.assert_allclose(gd.cpu().numpy(), od, rtol=1e-5)
    # the merged list is sorted by (dist, global id) and every id belongs to its shard range
    gi = gi.cpu().numpy()
    assert ((gi >= 0) & (gi < S * N_SHARD)).all()
