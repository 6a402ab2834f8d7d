"""P_max sweep with the oracle (SURVEY.md 8(c) "P_max value": never given by the paper; sweep
{0, 0.2, 0.5, 1, 2, 5} per config before GPU timing) plus graph reachability.

For each P_max: quantizer from the oracle, graph from the host builder (Alg1 l.17-18 adaptation),
then (a) layer-0 reachability from the entry point (BFS), (b) the quantizer's own ceiling: recall
of the exact top-k by d^q over the whole base (no graph), (c) recall of the AQR search (oracle) at
the given ef with a full re-rank, and (d) of the FP32-HNSW search on the same graph.

  python tools/pmax_sweep.py --config C1 --ef 512,1536 [--scale 1.0] [--nq 100]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2602_21600_b200 import graph as G  # noqa: E402


def reach(g):
    n = g.adj0.shape[0]
    seen = np.zeros(n, bool)
    seen[g.entry_point] = True
    front = np.array([g.entry_point])
    while len(front):
        nb = g.adj0[front].ravel()
        nb = np.unique(nb[nb >= 0])
        nb = nb[~seen[nb]]
        seen[nb] = True
        front = nb
    return float(seen.mean())


def recall(ids, gt):
    k = gt.shape[1]
    return float(np.mean([len(set(a) & set(b)) / k for a, b in zip(ids, gt)]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--ef", default="512,1536")
    ap.add_argument("--pmax", default="0,0.2,0.5,1,2,5")
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    w = synth.gen_config(args.config, scale=args.scale, nq=args.nq)
    k = w.k
    sample = synth.density_sample(len(w.x), seed=w.seed, cfg=args.config)
    gt, _ = oracle.bruteforce(w.x, w.q, k, w.metric)
    rho = oracle.density(w.x, sample)
    delta = oracle.delta(rho)
    eta = G.eta_of(G.density_weights(w.x[sample], rho))
    for pm in [float(v) for v in args.pmax.split(",")]:
        t0 = time.time()
        quant = oracle.train(w.x, sample, p_max=pm, delta_override=delta)
        codes = oracle.encode(w.x, quant)
        M, efc = G.adapt_params(w.M0, w.efc0, quant.delta, eta)
        g = G.build_hnsw(codes, M, efc, synth.level_draws(len(w.x), seed=w.seed, cfg=args.config), args.threads,
                         flags=1)
        ix = oracle.Index(w.x, codes, quant, g, w.metric)
        qc = oracle.encode(w.q, quant)
        bq, _ = oracle.bruteforce_dq(codes, w.x.shape[1], qc, k)
        row = dict(config=args.config, n=len(w.x), p_max=pm, delta=round(quant.delta, 4), M=M, efc=efc,
                   reach_layer0=round(reach(g), 5), dq_bruteforce_recall=round(recall(bq, gt), 4))
        for ef in [int(e) for e in args.ef.split(",")]:
            m = oracle.ef_mapping(ef, k)
            m["n_rerank"] = m["n_coarse"]
            ids, _ = oracle.search(ix, w.q, k, early_term=False, **m)
            fids, _ = oracle.search(ix, w.q, k, ef=max(ef, k), n_coarse=k, n_rerank=k, traversal="fp32")
            row[f"aqr_full_ef{ef}"] = round(recall(ids, gt), 4)
            row[f"fp32_ef{ef}"] = round(recall(fids, gt), 4)
        row["s"] = round(time.time() - t0, 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
