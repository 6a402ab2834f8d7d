"""Parameter sensitivity of the search (the paper's Table 3 presets and Fig. 3
axes): for each Table 3 preset (N_c, N_rerank, tau_gap, tau_ratio, m_ef) and an ef grid,
recall@10 (tie-aware), QPS of one aqr_search launch over the config's queries, the
early-termination rate and the mean exact re-rank depth.  One JSON line.

  python tools/sensitivity.py --config C2 --ef 256,384,512,784
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# Table 3: target recall band -> (N_c, N_rerank, tau_gap, tau_ratio, m_ef)
PRESETS = {"0.85-0.90": (35, 12, 0.020, 1.015, 2), "0.90-0.95": (45, 16, 0.015, 1.012, 2),
           "0.95-0.97": (55, 20, 0.012, 1.010, 3), "0.97+": (70, 28, 0.010, 1.008, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--ef", default="256,384,512,784")
    args = ap.parse_args()
    import torch
    import bench
    import synth
    import paper_2602_21600_b200 as aqr
    from paper_2602_21600_b200 import evaluate as E

    torch.cuda.set_device(0)
    w = synth.gen_config(args.config, scale=args.scale)
    x, codes, quant, g, ix, info = bench.build_index(w, args.config, 0, 1, 0)
    q = torch.from_numpy(w.q).cuda()
    gt_ids, gt_d = E.ground_truth(x, q, w.k, w.metric)
    rows = []
    for name, (nc0, nr0, tg, tr, m_ef) in PRESETS.items():
        for ef in [int(v) for v in args.ef.split(",")]:
            # the preset's (N_c, N_rerank) with ef scaled by m_ef (ef = N_c x m_ef); N_c
            # follows ef when ef / m_ef exceeds the preset's value (R13)
            nc = max(w.k, max(nc0, ef // m_ef))
            p = aqr.make_params(w.k, max(ef, nc), nc, min(max(w.k, nr0), nc), tg, tr, True)
            s = aqr.Searcher(ix, len(q), p)
            s.run(q)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.run(q)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            ids = s.ids.clone()
            ed = E.exact_dist(x, q, ids, w.metric).cpu().numpy()
            rec = E.recall(ids.cpu().numpy(), gt_ids, ed, gt_d, w.k)[1]
            s.totals.zero_()
            s.run(q, stats=True)
            torch.cuda.synchronize()
            t = s.totals.cpu().numpy() / len(q)
            r = dict(preset=name, ef=max(ef, nc), n_coarse=nc, n_rerank=p.n_rerank, tau_gap=tg, tau_ratio=tr, m_ef=m_ef,
                     recall=round(rec, 4), qps=round(len(q) / ms * 1e3, 1), et_rate=round(float(t[8]), 4),
                     depth=round(float(t[7]), 2))
            rows.append(r)
            print(json.dumps(r), file=sys.stderr, flush=True)
    print(json.dumps({"config": args.config, "index": {k: info[k] for k in ("M", "efc", "layout")}, "rows": rows}))


if __name__ == "__main__":
    main()
