"""Search latency on one GPU (the paper reports P50/P99 query latency on CPU,
Fig. 4).  Per batch size: one aqr_search launch per batch with CUDA events around each
launch (P50/P99 over reps), plus per-query latency inside one batch from the kernel's own
%globaltimer stamps (aqr_debug.t_ns): the service time of each query on its warp and its
completion time from the batch's first query start.  Prints one JSON line.

  python tools/latency.py --config C2 --ef 784 --batches 1,32,1024,10000 --reps 50
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--ef", type=int, default=784)
    ap.add_argument("--batches", default="1,32,1024,10000")
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    import torch
    import bench
    import synth
    import paper_2602_21600_b200 as aqr

    torch.cuda.set_device(0)
    w = synth.gen_config(args.config, scale=args.scale)
    x, codes, quant, g, ix, info = bench.build_index(w, args.config, 0, 1, 0)
    qall = torch.from_numpy(w.q).cuda()
    m = aqr.ef_mapping(args.ef, w.k)
    rng = np.random.default_rng(7)
    out = {"config": args.config, "ef": m["ef"], "n_coarse": m["n_coarse"], "n_rerank": m["n_rerank"],
           "index": {k: info[k] for k in ("M", "efc", "layout")}, "batches": []}
    for b in [int(v) for v in args.batches.split(",")]:
        b = min(b, len(w.q))
        s = aqr.Searcher(ix, b, aqr.make_params(w.k, **m))
        times = []
        for r in range(args.reps + 3):
            idx = torch.from_numpy(np.sort(rng.choice(len(w.q), b, replace=False))).cuda()
            qb = qall.index_select(0, idx).contiguous()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.run(qb)
            e1.record()
            torch.cuda.synchronize()
            if r >= 3:
                times.append(e0.elapsed_time(e1))
        t = np.array(times)
        # per-query latency inside the batch (aqr_debug.t_ns, %globaltimer): service time of each
        # query on its warp, and completion time from the batch's first query start
        s.run(qb, timing=True)
        torch.cuda.synchronize()
        tn = s.t_ns[:b].cpu().numpy().astype(np.float64)
        svc = (tn[:, 1] - tn[:, 0]) / 1e6
        done = (tn[:, 1] - tn[:, 0].min()) / 1e6
        out["batches"].append({"batch": b, "p50_ms": round(float(np.percentile(t, 50)), 4),
                               "p99_ms": round(float(np.percentile(t, 99)), 4),
                               "qps_p50": round(b / (np.percentile(t, 50) / 1e3), 1),
                               "query_service_ms": {"p50": round(float(np.percentile(svc, 50)), 4),
                                                    "p99": round(float(np.percentile(svc, 99)), 4),
                                                    "max": round(float(svc.max()), 4)},
                               "query_completion_ms": {"p50": round(float(np.percentile(done, 50)), 4),
                                                       "p99": round(float(np.percentile(done, 99)), 4),
                                                       "max": round(float(done.max()), 4)}})
        print(json.dumps(out["batches"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
