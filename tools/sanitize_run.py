"""A short end-to-end run of every kernel behind include/aqr.h for compute-sanitizer:
encode (training + pack), upload (GATHER and INLINE), search in each kernel configuration the tests
cover (AQR / FP32 traversal, one warp or a cooperative CTA per query, no visited set / shared-memory
hash / global bitmap, 128-d and 960-d rows, union assembly), the split re-rank and the shard merge, on small seeded inputs.  Checks the
results against the oracle so a silent corruption fails the run.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2602_21600_b200 as aqr  # noqa: E402
from tests._cases import case  # noqa: E402


def run(name, layouts=("gather", "inline"), vbits=(-1, 12, -2), traversals=("aqr", "fp32"), nq=8):
    c = case(name)
    x = torch.from_numpy(c.w.x).cuda()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(c.sample).cuda(), p_max=5.0,
                              delta_override=c.delta_override)
    torch.cuda.synchronize()
    assert np.array_equal(codes.cpu().numpy(), c.codes)
    q = np.ascontiguousarray(c.w.q[:nq])
    qd = torch.from_numpy(q).cuda()
    k = c.w.k
    p = dict(k=k, **oracle.ef_mapping(48, k))
    o_ids, _ = oracle.search(c.ix, q, **p)
    n_runs = 0
    for layout in layouts:
        ix = aqr.upload_index(codes, x, quant, c.graph, metric=c.w.metric, layout=layout)
        for tr in traversals:
            for vb in vbits:
                if layout == "inline" and vb not in (0, -1) and tr == "aqr":
                    continue
                # the cooperative kernel (4 warps per query) for AQR searches on the GATHER layout
                for wpq in ((1, 4) if (tr == "aqr" and layout == "gather") else (1,)):
                    ids, d, t = aqr.search(ix, qd, trace=True, visited_bits=vb, traversal=tr, warps_per_query=wpq, **p)
                    torch.cuda.synchronize()
                    if tr == "aqr":
                        assert np.array_equal(ids.cpu().numpy(), o_ids), (name, layout, vb, wpq)
                    n_runs += 1
        ids_u, _ = aqr.search(ix, qd, assemble_mode=1, **p)
        ids2, _ = aqr.rerank(ix, qd, t["coarse_ids"], k, p["n_rerank"])
        torch.cuda.synchronize()
        ix.free()
    dd = torch.rand(4, nq, k, device="cuda").sort(-1).values
    ii = torch.arange(4 * nq * k, dtype=torch.int32, device="cuda").reshape(4, nq, k)
    aqr.merge_topk(dd, ii)
    torch.cuda.synchronize()
    print(f"{name}: {n_runs} searches + union + rerank + merge ok", flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for nm in ["tiny7", "tiny33", "tiny100ip", "grid", "c4slice", "c1small"]:
        run(nm)
    print("sanitize_run ok")
