"""A/B timing of compile-time kernel variants (libaqr_<name>.so built by build.build_variant) on one
index in one process.  Every variant must return bit-identical ids (the visit order is fixed by
the method); the script asserts it.

  python tools/perf.py --config C2 --ef 896 --variants base,rows8,nopf [--layout gather]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_21600_b200 as aqr  # noqa: E402
from paper_2602_21600_b200 import build as B  # noqa: E402


def load(path):
    L = C.CDLL(path)
    L.aqr_last_error.restype = C.c_char_p
    L.aqr_version.restype = C.c_char_p
    L.aqr_index_device_bytes.restype = C.c_size_t
    L.aqr_search_workspace_size.restype = C.c_size_t
    L.aqr_index_layout.restype = C.c_int32
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--ef", default="896")
    ap.add_argument("--variants", default="base")
    ap.add_argument("--layout", default="gather")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--vbits", type=int, default=0)
    ap.add_argument("--wpq", default="0", help="warps_per_query values to time, e.g. 1,4")
    args = ap.parse_args()
    import torch
    import bench
    import synth
    from paper_2602_21600_b200 import evaluate as E

    torch.cuda.set_device(0)
    w = synth.gen_config(args.config, scale=args.scale, nq=args.nq)
    bench.LAYOUT = args.layout
    x, codes, quant, g, ix0, info = bench.build_index(w, args.config, 0, 1, 0)
    ix0.free()
    q = torch.from_numpy(w.q).cuda()
    gt_ids, gt_d = E.ground_truth(x, q, w.k, w.metric)
    out = []
    ref_ids = {}
    for name in args.variants.split(","):
        path = aqr.lib_path() if name == "default" else os.path.join(B.PKG, f"libaqr_{name}.so")
        aqr._lib = load(path)
        ix = aqr.upload_index(codes, x, quant, g, metric=w.metric, layout=args.layout)
        for ef, wpq in [(int(e), int(g)) for e in args.ef.split(",") for g in args.wpq.split(",")]:
            m = aqr.ef_mapping(ef, w.k)
            s = aqr.Searcher(ix, len(q), aqr.make_params(w.k, **m, visited_bits=args.vbits, warps_per_query=wpq))
            s.run(q)
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
            if ef in ref_ids:
                assert np.array_equal(ids, ref_ids[ef]), f"variant {name} changed the results at ef={ef}"
            else:
                ref_ids[ef] = ids
            ed = E.exact_dist(x, q, s.ids, w.metric).cpu().numpy()
            rec = E.recall(ids, gt_ids, ed, gt_d, w.k)[1]
            r = dict(variant=name, ef=ef, wpq=wpq, ms=round(ms, 3), qps=round(len(q) / ms * 1e3, 1), recall=round(rec, 4),
                     layout=ix.layout)
            out.append(r)
            print(json.dumps(r), flush=True)
        ix.free()
    print(json.dumps({"summary": out, "index": info}))


if __name__ == "__main__":
    main()
