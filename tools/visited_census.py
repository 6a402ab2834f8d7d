"""Visited-set census on one index: for each visited_bits setting, the search time (CUDA events)
and the per-query counters (layer-0 neighbour ids seen, evaluations scored, W insertions) from a
traced run.  The exact bitmap (-2) gives the distinct count; -1 scores every neighbour; a
direct-mapped shared-memory table of 2^b slots (b >= 6) sits in between (R15).

  python tools/visited_census.py --config C5 --ef 128 --vbits=-1,9,10,11,12,-2
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_21600_b200 as aqr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--ef", type=int, default=128)
    ap.add_argument("--vbits", default="-1,10,12,-2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--trace-nq", type=int, default=2000)
    args = ap.parse_args()
    import torch
    import bench
    import synth

    torch.cuda.set_device(0)
    w = synth.gen_config(args.config, scale=args.scale, nq=args.nq)
    x, codes, quant, g, ix, info = bench.build_index(w, args.config, 0, 1, 0)
    q = torch.from_numpy(w.q).cuda()
    m = aqr.ef_mapping(args.ef, w.k)
    ref = None
    for vb in [int(v) for v in args.vbits.split(",")]:
        s = aqr.Searcher(ix, len(q), aqr.make_params(w.k, **m, visited_bits=vb))
        s.run(q)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            s.run(q)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        ids = s.ids.cpu().numpy()
        same = None if ref is None else bool(np.array_equal(ids, ref))
        ref = ids if ref is None else ref
        nt = min(args.trace_nq, len(q))
        _, _, tr = aqr.search(ix, q[:nt], w.k, **m, visited_bits=vb, trace=True)
        c = tr["counters"].double().mean(0).cpu().numpy()
        r = dict(config=args.config, ef=args.ef, visited_bits=vb, ms=round(ms, 3),
                 qps=round(len(q) / ms * 1e3, 1), ids_equal_first=same, expansions=round(c[0], 1),
                 deg_sum=round(c[1], 1), scored=round(c[2], 1), below_thr=round(c[11], 1),
                 w_inserts=round(c[12], 1))
        print(json.dumps(r), flush=True)
    print(json.dumps({"index": info}, default=str)[:2000])


if __name__ == "__main__":
    main()
