"""Index build time (Table 2 analogue): the GPU build
(aqr_build_graph) against the host builder (csrc/hnsw_build.cpp, all host threads) on the same
codes and parameters, with a byte-for-byte comparison of the two graphs.

  python tools/build_time.py --config C2 [--no-host] [--scale 1.0]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-host", action="store_true")
    args = ap.parse_args()
    import torch
    import bench
    import synth
    import paper_2602_21600_b200 as aqr
    from paper_2602_21600_b200 import graph as G
    torch.cuda.set_device(0)
    cfg = args.config
    w = synth.gen_config(cfg, scale=args.scale, nq=10)
    x = torch.from_numpy(w.x).cuda()
    samp = synth.density_sample(len(w.x), seed=w.seed, cfg=cfg)
    t0 = time.time()
    codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(samp).cuda(), p_max=bench.P_MAX[cfg], want_rho=True)
    torch.cuda.synchronize()
    t_enc = time.time() - t0
    eta = G.eta_of(G.density_weights(w.x[samp], quant.rho.cpu().numpy()))
    M, efc = G.adapt_params(w.M0, w.efc0, quant.delta, eta)
    lu = synth.level_draws(len(w.x), seed=w.seed, cfg=cfg)
    G.build_hnsw_gpu(codes[:2048], w.x.shape[1], M, efc, lu[:2048], flags=bench.BUILD_FLAGS)  # warm-up
    torch.cuda.synchronize()
    t0 = time.time()
    gg = G.build_hnsw_gpu(codes, w.x.shape[1], M, efc, lu, flags=bench.BUILD_FLAGS)
    t_gpu = time.time() - t0
    row = dict(config=cfg, n=len(w.x), d=w.x.shape[1], M=M, efc=efc, encode_s=round(t_enc, 2),
               gpu_build_s=round(t_gpu, 2), max_level=gg.max_level, host_threads=os.cpu_count())
    if not args.no_host:
        t0 = time.time()
        hg = G.build_hnsw(codes.cpu().numpy(), M, efc, lu, 0, flags=bench.BUILD_FLAGS)
        row["host_build_s"] = round(time.time() - t0, 2)
        row["speedup"] = round(row["host_build_s"] / t_gpu, 1)
        row["graphs_identical"] = bool(np.array_equal(hg.adj0, gg.adj0) and np.array_equal(hg.adj_upper, gg.adj_upper)
                                       and (hg.entry_point, hg.max_level) == (gg.entry_point, gg.max_level))
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
