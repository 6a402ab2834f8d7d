"""bench.py -- QPS at recall@10 >= 0.98 of the B200-native AQR-HNSW search (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--config C2] [--ef auto|E] [--impl aqr|reference]
  (N > 1: launched with torch.distributed.run, one process per GPU, NCCL)

A "step" is one pass of the whole hot path (aqr_search: query quantization, greedy descent,
layer-0 beam, Stage 2, early termination, Stage 3, assembly) over this rank's slice of the
query batch.  C1-C4 replicate the index on every GPU and split the queries (weak scaling:
each rank searches the full 10k query set, so per-GPU work is fixed as N grows; no data-path
collective).  Index construction (generation, GPU encode, host HNSW build, upload) happens
before the timed region.

The JSON line carries `roofline` (the search kernel against the measured HBM copy bandwidth,
algorithmic bytes per DESIGN.md "Bytes per query"), `cpu_baseline` (the CPU oracle on a
bounded query sample, rank 0, N = 1), `e2e` (through the public API with host buffers and
the H2D/D2H copies inside the timed region) and `clocks` (nvidia-smi during the timed region).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EF_GRID = [16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512, 640, 768, 896, 1024, 1280, 1536, 2048, 3072, 4096, 6144, 8192]
# per-config quantizer window P_max (never given by the paper; R4) and the
# fixed HNSW construction inputs of BASELINE.json
P_MAX = {"C1": 0.2, "C2": 0.2, "C3": 0.0, "C4": 0.2, "C5": 5.0}
TARGET_RECALL = 0.98
# the operating point our arm reports (smallest ef with recall@10 >= 0.98 and its re-rank mapping,
# measured: profiles/r02/bench_c*.json): the reference arm (the oracle) is timed on the same point
AT_TARGET = {"C1": (64, "exact"), "C2": (784, "preset"), "C3": (5888, "exact"), "C4": (2480, "full"),
             "C5": (128, "preset")}
LAYOUT = "auto"
WJ_LITERAL = False  # --wj literal: Alg1 l.12 as printed (NEXT-4 variant; R16)
BUILDER = "gpu"  # --builder: the index build on the GPU (aqr_build_graph) or the host builder
BUILD_FLAGS = 1  # host builder: Malkov's keepPrunedConnections (R14)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------------------------
# distributed plumbing
# --------------------------------------------------------------------------------------------
def relaunch_if_needed(args):
    """--gpus N > 1 means N processes, one per GPU: when the script was not started by
    torch.distributed.run (no WORLD_SIZE), start it that way (rendezvous on 127.0.0.1) and return
    its exit code; when it was, WORLD_SIZE must equal N."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus <= 1:
            return None
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        log(f"[bench] --gpus {args.gpus}: relaunching under torch.distributed.run ({args.gpus} processes)")
        return subprocess.call(cmd)
    if int(world) != args.gpus:
        log(f"[bench] WORLD_SIZE={world} but --gpus {args.gpus}: refusing to run (they must agree)")
        return 2
    return None


def dist_init(n_gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"[bench] WORLD_SIZE={world} != --gpus {n_gpus}")
    if world > 1:
        # one process per GPU over NCCL.  AQR_DIST_BACKEND=gloo runs the same multi-rank code path
        # with several ranks sharing a device (a functional check of the N > 1 plumbing on a
        # one-GPU box; never a measurement: the ranks time-share the GPU)
        backend = os.environ.get("AQR_DIST_BACKEND", "nccl")
        dev = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # NCCL's own init lines (transport, NVLS)
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
        local = dev
        nccl_v = ".".join(map(str, torch.cuda.nccl.version())) if backend == "nccl" else "-"
        log(f"[bench] rank {rank}/{dist.get_world_size()} backend={dist.get_backend()} device=cuda:{dev} "
            f"({torch.cuda.get_device_name(dev)}) nccl={nccl_v} host_cpus={os.cpu_count()}")
        assert dist.get_world_size() == n_gpus
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor(np.asarray(v, dtype=np.float64), device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def bcast_np(a, world, rank, dtype):
    """Broadcast a host array from rank 0 (shape broadcast first)."""
    if world == 1:
        return a
    import torch
    import torch.distributed as dist
    shp = torch.zeros(4, dtype=torch.int64, device="cuda")
    if rank == 0:
        s = list(a.shape) + [0] * (4 - a.ndim)
        shp[:] = torch.tensor(s)
        shp[3] = a.ndim
    dist.broadcast(shp, 0)
    nd = int(shp[3].item())
    shape = tuple(int(v) for v in shp[:nd].tolist())
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda() if rank == 0 else torch.empty(shape, dtype=dtype, device="cuda")
    dist.broadcast(t, 0)
    return t.cpu().numpy()


# --------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# --------------------------------------------------------------------------------------------
class Clocks:
    """SM clocks and clock-event reasons sampled DURING the timed region: NVML polled from a thread
    every 5 ms (a sample is taken at start() and at stop(), so even a ~100 ms region has samples);
    nvidia-smi -lms 100 if NVML is unavailable."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clock-event reason bits (nvml.h)
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.p = None
        self.nv = None
        self.lines = []
        self.samples = []

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.gpu).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def _sample(self):
        nv, h = self.nv
        self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetCurrentClocksEventReasons(h)))

    def _poll(self):
        while not self.done.is_set():
            try:
                self._sample()
            except Exception:
                return
            self.done.wait(0.005)

    def start(self):
        try:
            self.nv = self._handle()
            self._sample()
            self.done = threading.Event()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._rd, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5:  # the region starts once sampling runs
                time.sleep(0.01)
        except Exception:
            self.p = None

    def _rd(self):
        for ln in self.p.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.nv is not None:
            self.done.set()
            self.t.join(1)
            try:
                self._sample()
            except Exception:
                pass
            sm = [float(a) for a, _, _ in self.samples]
            mx = [float(b) for _, b, _ in self.samples]
            reasons = {nm for _, _, r in self.samples for nm, bit in self.BITS.items() if r & bit}
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        n0 = len(self.lines)
        t0 = time.time()
        while len(self.lines) == n0 and time.time() - t0 < 1:  # one sample at the region's end
            time.sleep(0.01)
        self.p.terminate()
        try:
            self.p.wait(2)
        except Exception:
            self.p.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


# --------------------------------------------------------------------------------------------
# workload + index construction (outside the timed region)
# --------------------------------------------------------------------------------------------
def make_workload(cfg, scale, nq):
    import synth
    return synth.gen_config(cfg, scale=scale, nq=nq)


def build_index(w, cfg, rank, world, threads, delta_override=None):
    import torch
    import synth
    import paper_2602_21600_b200 as aqr
    from paper_2602_21600_b200 import graph as G
    t0 = time.time()
    x = torch.from_numpy(w.x).cuda()
    sample_np = synth.density_sample(len(w.x), seed=w.seed, cfg=cfg)
    sample = torch.from_numpy(sample_np).cuda()
    codes, quant = aqr.encode(x, sample_idx=sample, p_max=P_MAX[cfg], want_rho=True, delta_override=delta_override)
    torch.cuda.synchronize()
    t_enc = time.time() - t0
    rho = quant.rho.cpu().numpy()
    wj = G.density_weights(w.x[sample_np], rho, literal=WJ_LITERAL)
    eta = G.eta_of(wj)
    M, efc = G.adapt_params(w.M0, w.efc0, quant.delta, eta)
    t1 = time.time()
    level_u = synth.level_draws(len(w.x), seed=w.seed, cfg=cfg)
    if BUILDER == "gpu":
        # the GPU index build (aqr_build_graph, NEXT-1): deterministic, so every rank builds the
        # same graph on its own GPU (byte-identical with the host builder and the oracle)
        g = G.build_hnsw_gpu(codes, w.x.shape[1], M, efc, level_u, flags=BUILD_FLAGS)
    else:
        if rank == 0:
            g = G.build_hnsw(codes.cpu().numpy(), M, efc, level_u, threads, flags=BUILD_FLAGS)
            arrs = [g.levels, g.upper_off, g.adj0, g.adj_upper, np.array([g.entry_point, g.max_level], np.int64)]
        else:
            arrs = [None] * 5
        if world > 1:
            dts = [torch.int32, torch.int64, torch.int32, torch.int32, torch.int64]
            arrs = [bcast_np(a, world, rank, dt) for a, dt in zip(arrs, dts)]
            g = G.Graph(M, efc, arrs[0], arrs[1], arrs[2], arrs[3], int(arrs[4][0]), int(arrs[4][1]))
    t_build = time.time() - t1
    ix = aqr.upload_index(codes, x, quant, g, metric=w.metric, layout=LAYOUT)
    reach = layer0_reach(g) if rank == 0 else None
    info = dict(layout=ix.layout, reach_layer0=reach, builder=BUILDER, build_flags=BUILD_FLAGS, wj="literal" if WJ_LITERAL else "spec", delta=quant.delta, eta=eta, M=M, efc=efc, p_max=P_MAX[cfg], p_low=quant.p_low, p_high=quant.p_high,
                encode_s=round(t_enc, 2), build_s=round(t_build, 2), max_level=g.max_level,
                index_bytes=ix.device_bytes())
    return x, codes, quant, g, ix, info


def layer0_reach(g):
    """Share of the nodes reachable from the entry point on layer 0 (BFS; SPEC S:431's >= 99%): a
    recall ceiling of the graph itself, whatever the search does."""
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
    return round(float(seen.mean()), 6)


def bytes_per_query(tot, nq, d, k, distinct_ratio=1.0, traversal="aqr"):
    """Algorithmic bytes from the kernel counters:
    query 4d + adjacency 4(deg+1) per expansion (all layers) + d per DISTINCT code evaluation
    (all layers) + N_c d (Stage 2 re-read) + 4d per exact re-rank + 8k output.  The kernel
    counts every neighbour it scores (it keeps no exact visited set); `distinct_ratio` = distinct
    evaluations / neighbours scored, measured exactly by the oracle (same visit order) on a query
    sample, converts that count to the algorithmic one."""
    exp, deg, ev, uexp, udeg, uev, nc, depth, et, na, fails = [float(v) for v in tot[:11]]
    if traversal == "fp32":  # the baseline reads a 4d-byte fp32 row per distinct evaluation, no re-rank
        b = (4 * d * nq + 4 * (deg + exp) + 4 * (udeg + uexp) + 4 * d * ((ev - fails) * distinct_ratio + uev)
             + 8 * k * nq)
        return b / nq
    b = (4 * d * nq + 4 * (deg + exp) + 4 * (udeg + uexp) + d * ((ev - fails) * distinct_ratio + uev) + d * nc
         + 4 * d * depth + 8 * k * nq)
    return b / nq


def sector_bytes_per_query(tot, nq, d, k, distinct_ratio=1.0, traversal="aqr"):
    """bytes_per_query at 32-byte sector granularity: each row read rounded up to
    whole sectors (C3's 100-byte codes occupy 128 B); adjacency rows rounded at the mean degree."""
    def sec(b):
        return 32.0 * math.ceil(b / 32.0)
    exp, deg, ev, uexp, udeg, uev, nc, depth, et, na, fails = [float(v) for v in tot[:11]]
    adj = exp * sec(4 * (deg / max(exp, 1.0) + 1)) + uexp * sec(4 * (udeg / max(uexp, 1.0) + 1))
    evals = (ev - fails) * distinct_ratio + uev
    if traversal == "fp32":
        b = sec(4 * d) * nq + adj + sec(4 * d) * evals + 8 * k * nq
    else:
        b = sec(4 * d) * nq + adj + sec(d) * (evals + nc) + sec(4 * d) * depth + 8 * k * nq
    return b / nq


def oracle_index(w, cfg, codes, g, delta_override=float("nan")):
    """The oracle trains its own quantizer and encodes the base itself (full-size parity check
    of aqr_encode: codes compared byte for byte), then searches the same graph."""
    import oracle
    import synth
    t0 = time.time()
    sample = synth.density_sample(len(w.x), seed=w.seed, cfg=cfg)
    o_quant = oracle.train(w.x, sample, p_max=P_MAX[cfg], delta_override=delta_override)
    o_codes = oracle.encode(w.x, o_quant)
    codes_equal = bool(np.array_equal(o_codes, codes.cpu().numpy()))
    return oracle.Index(w.x, o_codes, o_quant, g, w.metric), codes_equal, time.time() - t0


def distinct_ratio_from_oracle(oix, w, m, k, n_sample=256, traversal="aqr"):
    import oracle
    _, _, tr = oracle.search(oix, w.q[:n_sample], k, trace=True, exp_cap=1, traversal=traversal, **m)
    cnt = tr["counters"].sum(0)
    # layer-0 distinct evaluations / layer-0 neighbours seen (oracle counters 2 and 1)
    return float(cnt[2]) / max(float(cnt[1]), 1.0), int(len(w.q[:n_sample]))


# --------------------------------------------------------------------------------------------
# the AQR arm
# --------------------------------------------------------------------------------------------
def run_aqr(args):
    import torch
    import paper_2602_21600_b200 as aqr
    from paper_2602_21600_b200 import evaluate as E

    rank, world, local = dist_init(args.gpus)
    cfg = args.config
    w = make_workload(cfg, args.scale, args.nq)
    k = w.k
    nq = len(w.q)
    from paper_2602_21600_b200 import parallel as P
    if args.scaling == "weak":
        # world x nq distinct queries, nq per rank (rank 0: the config's set; others: stream 3)
        src, lo, hi = P.weak_block(nq, world, rank)
        if src == "config":
            q_host = np.ascontiguousarray(w.q)
        else:
            import synth
            q_host = np.ascontiguousarray(synth.gen_query_stream(cfg, hi, seed=w.seed)[lo:hi])
        q_src = f"{src} rows [{lo}, {hi})"
    else:
        lo, hi = P.query_range(nq, world, rank)  # strong scaling: one batch split
        q_host = np.ascontiguousarray(w.q[lo:hi])
        q_src = f"config rows [{lo}, {hi})"
    if rank == 0:
        log(f"[bench] {args.scaling} scaling over {world} rank(s); rank 0 queries: {q_src}")
    q = torch.from_numpy(q_host).cuda()
    sq8 = args.traversal == "sq8"
    x, codes, quant, g, ix, info = build_index(w, cfg, rank, world, args.threads, 0.0 if sq8 else None)
    if rank == 0:
        log(f"[bench] {cfg} n={len(w.x)} d={w.x.shape[1]} nq={nq} index: {info}")

    # ground truth for this rank's queries, then the ef sweep (recall summed over ranks)
    gt_ids, gt_d = E.ground_truth(x, q, k, w.metric)
    sweep = []
    chosen = None
    grid = EF_GRID if args.ef == "auto" else [int(args.ef)]

    def mapping(ef, mode):
        # "preset": Table 3 "0.97+" (R13); "full": the same N_c with every C entry re-ranked
        # exactly (N_rerank = N_c) -- the Fig. 3 knob for data where d^q / d^a order is noisy (R20);
        # "exact": full with the early-termination thresholds at infinity (R26), so a
        # d^a gap can no longer cut the exact re-rank to k
        if args.traversal == "fp32":  # the baseline: W's first k are the result
            return dict(ef=max(ef, k), n_coarse=k, n_rerank=k)
        mm = mode_mapping(aqr.ef_mapping, ef, k, mode, sq8)
        if args.tau_spread != float("inf") and not sq8:  # adaptive depth (NEXT-4, R27)
            mm["tau_spread"] = args.tau_spread
        return mm

    def measure(ef, mode):
        m = mapping(ef, mode)
        p = aqr.make_params(k, **m, visited_bits=args.vbits[0], traversal=args.kt)
        s = aqr.Searcher(ix, len(q), p)
        s.run(q)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        s.run(q)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        ids = s.ids.clone()
        ed = E.exact_dist(x, q, ids, w.metric).cpu().numpy()
        ov, ta = E.recall(ids.cpu().numpy(), gt_ids, ed, gt_d, k)
        tot = allreduce_sum([ov * len(q), ta * len(q), len(q)], world)
        ms_max = allreduce_max(ms, world)
        r = dict(ef=ef, rerank=mode, n_coarse=m["n_coarse"], n_rerank=m["n_rerank"],
                 recall=round(tot[1] / tot[2], 4), recall_id=round(tot[0] / tot[2], 4),
                 qps=round(float(tot[2]) / (ms_max / 1e3), 1))
        if rank == 0:
            log(f"[bench] sweep {r}")
        return r

    best = None  # (qps, ef, mode)
    for mode in args.rerank.split(","):
        chosen = None
        prev = None
        for ef in grid:
            r = measure(ef, mode)
            sweep.append(r)
            if r["recall"] >= TARGET_RECALL and chosen is None:
                chosen = ef
                if args.ef == "auto" and not args.full_sweep:
                    break
            if chosen is None:
                prev = ef
        if chosen is not None and prev is not None and args.ef == "auto":
            # refine: the smallest ef (multiple of 16) between the last failing grid point and the
            # first passing one whose recall@10 >= target (recall is monotone in ef up to noise)
            lo, hi = prev, chosen
            while hi - lo > 16:
                mid = (lo + hi) // 2 // 16 * 16
                if mid <= lo:
                    break
                r = measure(mid, mode)
                sweep.append(r)
                if r["recall"] >= TARGET_RECALL:
                    hi = mid
                else:
                    lo = mid
            chosen = hi
        if chosen is not None:
            qps = max(z["qps"] for z in sweep if z["ef"] == chosen and z["rerank"] == mode)
            if best is None or qps > best[0]:
                best = (qps, chosen, mode)
    sweep.sort(key=lambda z: (z["rerank"], z["ef"]))
    target_met = best is not None
    if best is None:
        # no point reached the target: report the highest-recall point of the sweep (the ceiling)
        top = max(sweep, key=lambda z: (z["recall"], z["qps"]))
        best = (top["qps"], top["ef"], top["rerank"])
    chosen, chosen_mode = best[1], best[2]
    m = mapping(chosen, chosen_mode)
    vb_results = []
    best_vb, best_ms = 0, float("inf")
    for vb in args.vbits:
        p = aqr.make_params(k, **m, visited_bits=vb, traversal=args.kt)
        s = aqr.Searcher(ix, len(q), p)
        s.run(q)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(3):
            s.run(q)
        ev1.record()
        torch.cuda.synchronize()
        ms = allreduce_max(ev0.elapsed_time(ev1) / 3, world)
        vb_results.append(dict(visited_bits=vb, ms=round(ms, 3)))
        if ms < best_ms:
            best_vb, best_ms = vb, ms
    if rank == 0 and len(args.vbits) > 1:
        log(f"[bench] visited_bits sweep {vb_results} -> {best_vb}")
    p = aqr.make_params(k, **m, visited_bits=best_vb, traversal=args.kt)
    s = aqr.Searcher(ix, len(q), p)
    wpq_plan = aqr.search_plan(ix, len(q), p)  # 1: search_kernel (a warp per query), 4: coop_kernel
    # counters for the roofline (separate, untimed run with the stats path)
    s.totals.zero_()
    s.run(q, stats=True)
    torch.cuda.synchronize()
    tot_counters = s.totals.cpu().numpy()
    oix, codes_equal, t_otrain = (None, None, 0.0)
    ratio, n_ratio = 1.0, 0
    if rank == 0 and not args.no_oracle:
        oix, codes_equal, t_otrain = oracle_index(w, cfg, codes, g, 0.0 if sq8 else float("nan"))
        ratio, n_ratio = distinct_ratio_from_oracle(oix, w, m, k, traversal=args.kt)
    ratio = float(allreduce_sum([ratio if rank == 0 else 0.0], world)[0]) if world > 1 else ratio
    queries_all = int(allreduce_sum([len(q)], world)[0]) if world > 1 else len(q)
    if best_vb != -1 and best_vb != 0:
        ratio = 1.0  # a visited set: the kernel's evaluation count is already the distinct one
    bq = bytes_per_query(tot_counters, len(q), w.x.shape[1], k, ratio, args.kt)
    bq_sector = sector_bytes_per_query(tot_counters, len(q), w.x.shape[1], k, ratio, args.kt)

    # ---- the search kernel alone: isolated launches on one stream, events around each (the
    # roofline's kernel time) ----
    stream = torch.cuda.current_stream()
    s.run(q)
    torch.cuda.synchronize()
    iso = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(max(3, args.steps))]
    for a, b in iso:
        a.record(stream)
        s.run(q)
        b.record(stream)
    torch.cuda.synchronize()
    launch_ms = float(np.mean([a.elapsed_time(b) for a, b in iso]))

    # ---- device-timed region: W warm-up steps, then K steps bracketed by barrier + sync.  Steps
    # are issued round-robin on P streams (--pipeline, default 2), each with its own Searcher
    # (outputs + workspace), so the persistent grid's tail of one step overlaps the start of the
    # next, as consecutive batches of a serving loop do; every step searches its whole batch ----
    P = max(1, args.pipeline)
    searchers = [s] + [aqr.Searcher(ix, len(q), p) for _ in range(P - 1)]
    streams = [torch.cuda.Stream() for _ in range(P)]

    def run_steps(nsteps, gate):
        for st in streams:
            st.wait_event(gate)
        for i in range(nsteps):
            searchers[i % P].run(q, stream=streams[i % P])
        for st in streams:
            stream.wait_stream(st)

    g0 = torch.cuda.Event()
    g0.record(stream)
    run_steps(args.warmup, g0)
    torch.cuda.synchronize()
    barrier(world)
    clocks = Clocks(local)
    clocks.start()
    barrier(world)
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    run_steps(args.steps, t_start)
    t_end.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    total_ms = allreduce_max(total_ms, world)
    # every step's results are the searchers' (identical queries -> identical results)
    for sx in searchers[1:]:
        assert torch.equal(sx.ids, s.ids), "pipelined searchers disagree"
    ms_per_step = total_ms / args.steps
    queries_per_step_all = queries_all  # distinct queries searched by all ranks in one step
    value = queries_per_step_all / (ms_per_step / 1e3)

    # ---- end to end through the public API: pinned host queries in, host results out ----
    qh = torch.from_numpy(q_host).pin_memory()
    ids_h = torch.empty((len(q), k), dtype=torch.int32).pin_memory()
    dist_h = torch.empty((len(q), k), dtype=torch.float32).pin_memory()
    qd = torch.empty_like(q)
    # per pipeline stream: its own device query buffer and pinned host outputs
    qds = [qd] + [torch.empty_like(q) for _ in range(P - 1)]
    outs_h = [(ids_h, dist_h)] + [(torch.empty_like(ids_h).pin_memory(), torch.empty_like(dist_h).pin_memory())
                                  for _ in range(P - 1)]

    def e2e_steps(nsteps, gate):
        for st in streams:
            st.wait_event(gate)
        for i in range(nsteps):
            j = i % P
            with torch.cuda.stream(streams[j]):
                qds[j].copy_(qh, non_blocking=True)
                searchers[j].run(qds[j], stream=streams[j])
                outs_h[j][0].copy_(searchers[j].ids, non_blocking=True)
                outs_h[j][1].copy_(searchers[j].dist, non_blocking=True)
        for st in streams:
            stream.wait_stream(st)

    g1 = torch.cuda.Event()
    g1.record(stream)
    e2e_steps(2 * P, g1)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_steps(args.steps, e0)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = allreduce_max(e0.elapsed_time(e1) / args.steps, world)
    e2e_val = queries_per_step_all / (e2e_ms / 1e3)
    h2d_all = int(allreduce_sum([q_host.nbytes], world)[0]) if world > 1 else int(q_host.nbytes)
    d2h_all = int(allreduce_sum([ids_h.numel() * 8], world)[0]) if world > 1 else int(ids_h.numel() * 8)

    # ---- optional steady-state stream: fresh queries, same index and parameters ----
    steady = None
    if args.stream > 0:
        import synth
        qs = torch.from_numpy(synth.gen_query_stream(cfg, args.stream)).cuda()
        ss = aqr.Searcher(ix, len(qs), p)
        ss.run(qs)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(3):
            ss.run(qs)
        s1.record(stream)
        torch.cuda.synchronize()
        sms = allreduce_max(s0.elapsed_time(s1) / 3, world)
        steady = {"queries_per_rank": len(qs), "qps": round(len(qs) * world / (sms / 1e3), 1),
                  "ms_per_launch": round(sms, 3), "note": "fresh queries (stream 3), same index / ef"}

    # ---- roofline of the dominant kernel (search_kernel: one launch per step) ----
    import json as _json
    peaks = {}
    try:
        peaks = _json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    bytes_launch = bq * len(q)
    achieved = bytes_launch / (launch_ms / 1e3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            tj = _json.load(open(tf))
            if tj.get("config") == cfg and tj.get("ef") == chosen and tj.get("nq") == len(q):
                traffic = tj.get("bytes_per_launch")
        except Exception:
            pass

    # ---- CPU oracle baseline: rank 0, N = 1, bounded query sample ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and oix is not None:
        cpu = cpu_baseline(w, oix, m, k, args.cpu_seconds, s, args.kt)
        cpu["codes_equal_full_size"] = codes_equal
        cpu["oracle_train_s"] = round(t_otrain, 1)

    if rank == 0:
        line = {
            "metric": "QPS at recall@10>=0.98" if target_met else
                      "QPS at the ceiling recall@10 (no ef in the sweep reached 0.98; see config.recall@10)",
            "target_met": target_met,
            "value": round(value, 1), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u8+int32+f32",
            "data": "synthetic (seeded, BASELINE.json config recipe; paper datasets unavailable)",
            "config": {"workload": f"{cfg}: {len(w.x)} x {w.x.shape[1]} {w.metric}, {nq} queries, k={k}",
                       "queries_per_step": queries_per_step_all,
                       "query_split": ("weak: world x nq distinct queries, nq per rank (rank 0 the config's set, "
                                       "ranks >= 1 synth stream 3)") if args.scaling == "weak"
                       else "strong: the config's nq split contiguously",
                       "ef": chosen, "n_coarse": m["n_coarse"], "n_rerank": m["n_rerank"],
                       "rerank": chosen_mode, "traversal": args.traversal,
                       "recall@10": next((z["recall"] for z in sweep if z["ef"] == chosen and z["rerank"] == chosen_mode),
                                         None),
                       "visited_bits": best_vb, "visited_bits_sweep": vb_results, "queries_per_rank": len(q),
                       "warps_per_query": wpq_plan,
                       "parallelism": f"replicated index, query-parallel over {world} GPU(s), no data-path collective",
                       "l2": "index (codes+adjacency+fp32) > 126 MB L2; no flush",
                       "pipeline": P, "pipeline_note": ("steps issued round-robin on this many CUDA streams, each "
                                                        "with its own outputs and workspace: one step's grid tail "
                                                        "overlaps the next step's start; roofline.kernel_ms is an "
                                                        "isolated single-stream launch"), **info},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "frac_pipelined": round(bytes_launch / (ms_per_step / 1e3) / 1e9 / peak, 4),
                         "limiter": ("below the HBM roofline the kernel is bound by per-warp dependent chains and "
                                     "issue (ncu: DRAM ~11% of peak, L2 hit ~78%, issue ~59% busy; "
                                     "profiles/r02/ncu_search_c2_s4final*.txt)"),
                         "bytes_per_query": round(bq, 1), "sector_bytes_per_query": round(bq_sector, 1),
                         "peak_source": peak_src,
                         "distinct_eval_ratio": round(ratio, 4), "distinct_ratio_sample": n_ratio,
                         "kernel": "coop_kernel" if wpq_plan == 4 else "search_kernel", "kernel_ms": round(launch_ms, 4)},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_val, 1), "unit": "queries/s",
                    "h2d_bytes_per_step": h2d_all, "d2h_bytes_per_step": d2h_all,
                    "note": "all ranks; pinned host queries in and ids + distances out inside the timed region"},
            "gpu_launches": args.steps,
            "ms_per_step_isolated": round(launch_ms, 4),
            "steady_state": steady,
            "lib": aqr.lib().aqr_version().decode(),  # "... src:<hash of the CUDA sources libaqr.so was built from>"
            "clocks": clk,
            "ef_sweep": sweep,
            "counters_per_query": {n: round(float(v) / len(q), 2) for n, v in zip(aqr.COUNTER_NAMES, tot_counters)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def cpu_model():
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_search_threads(oix, q, k, threads, traversal="aqr", **m):
    """The oracle as it stands, query-parallel: `threads` host threads each run the unchanged
    single-threaded C search on a contiguous slice (ctypes releases the GIL during the call), so
    the ids are those of one sequential run."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    if threads <= 1 or len(q) < 2:
        return oracle.search(oix, q, k, traversal=traversal, **m)
    cuts = np.linspace(0, len(q), min(threads, len(q)) + 1).astype(int)
    parts = [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    with ThreadPoolExecutor(len(parts)) as ex:
        outs = list(ex.map(lambda ab: oracle.search(oix, q[ab[0]:ab[1]], k, traversal=traversal, **m), parts))
    return np.concatenate([o[0] for o in outs]), np.concatenate([o[1] for o in outs])


def cpu_baseline(w, oix, m, k, seconds, searcher, traversal="aqr"):
    """The CPU oracle as it stands on a bounded sample of the same queries: query-parallel on all
    host cores (the reported value) and single-threaded beside it."""
    import oracle
    n_try = 8
    t0 = time.time()
    oracle.search(oix, w.q[:n_try], k, traversal=traversal, **m)
    per_q = (time.time() - t0) / n_try
    n_s = int(max(n_try, min(len(w.q), seconds / 2 / max(per_q, 1e-6))))
    t0 = time.time()
    o_ids, _ = oracle.search(oix, w.q[:n_s], k, traversal=traversal, **m)
    el = time.time() - t0
    cores = os.cpu_count() or 1
    n_a = int(min(len(w.q), max(cores, n_s * cores)))
    t0 = time.time()
    a_ids, _ = oracle_search_threads(oix, w.q[:n_a], k, cores, traversal=traversal, **m)
    el_a = time.time() - t0
    g_ids = searcher.ids[:n_a].cpu().numpy()
    same = bool(np.array_equal(a_ids[:n_s], o_ids))
    return {"value": round(n_a / el_a, 2), "unit": "queries/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"first {n_a} of {len(w.q)} queries, same graph/ef; the single-threaded C oracle run "
                      f"query-parallel on {cores} host threads ({el_a:.1f} s)",
            "single_core": {"value": round(n_s / el, 2), "cores": 1,
                            "sample": f"first {n_s} queries, one thread ({el:.1f} s)",
                            "ids_identical_to_parallel_run": same},
            "ids_equal_frac": round(float((a_ids == g_ids).all(1).mean()), 4)}


def cpu_baseline_sharded(keep0, q_host, searcher0, m, k, n_shards, seconds):
    """C5's cpu_baseline: the oracle as it stands on shard 0 (its own quantizer and codes, compared
    byte for byte with aqr_encode's; the same graph), a bounded query sample on all host threads.
    A CPU serving the whole job searches every shard, so the job-level value is the shard-0 rate
    divided by the number of shards (the merge is negligible beside it)."""
    import oracle
    import torch
    xs, samp, codes, g = keep0
    t0 = time.time()
    o_quant = oracle.train(xs, samp, p_max=P_MAX["C5"])
    o_codes = oracle.encode(xs, o_quant)
    codes_equal = bool(np.array_equal(o_codes, codes.cpu().numpy()))
    oix = oracle.Index(xs, o_codes, o_quant, g, "l2")
    prep = time.time() - t0
    cores = os.cpu_count() or 1
    t0 = time.time()
    oracle.search(oix, q_host[:4], k, **m)
    per_q = (time.time() - t0) / 4
    n_a = int(max(cores, min(len(q_host), seconds * cores / max(per_q, 1e-6))))
    t0 = time.time()
    a_ids, _ = oracle_search_threads(oix, q_host[:n_a], k, cores, **m)
    el = time.time() - t0
    searcher0.run(torch.from_numpy(q_host).cuda())
    torch.cuda.synchronize()
    g_ids = searcher0.ids[:n_a].cpu().numpy()  # shard 0: id_base 0
    return {"value": round(n_a / el / n_shards, 2), "unit": "queries/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"shard 0 of {n_shards}, first {n_a} of {len(q_host)} queries, same graph/ef, the single-threaded C "
                      f"oracle query-parallel on {cores} host threads ({el:.1f} s; training + encoding the shard "
                      f"{prep:.1f} s, untimed); value = shard-0 rate {n_a / el:.1f} / {n_shards} shards",
            "codes_equal_shard0": codes_equal,
            "ids_equal_frac": round(float((a_ids == g_ids).all(1).mean()), 4)}


# --------------------------------------------------------------------------------------------
# C5: the base sharded 8 ways; per-shard top-k merged locally, then over NCCL
# --------------------------------------------------------------------------------------------
def run_sharded(args):
    import torch
    import synth
    import paper_2602_21600_b200 as aqr
    from paper_2602_21600_b200 import evaluate as E
    from paper_2602_21600_b200 import graph as G
    from paper_2602_21600_b200 import parallel as P

    rank, world, local = dist_init(args.gpus)
    S = 8
    n_shard = max(1, int(round(1_250_000 * args.scale)))
    nq = args.nq or 10_000
    k = 100
    ef = 128 if args.ef == "auto" else int(args.ef)
    m = aqr.ef_mapping(ef, k)
    q_host = synth.gen_c5_queries(nq)  # every rank generates the same queries from the seed
    q = torch.from_numpy(q_host).cuda()
    mine = P.shards_of_rank(S, world, rank)
    threads = args.threads or max(1, (os.cpu_count() or 1) // min(world, 8))
    shards, infos = [], []
    gt_d_parts, gt_i_parts = [], []
    keep0 = None
    for s_ in mine:
        t0 = time.time()
        xs = synth.gen_c5_shard(s_, n_shard)
        x = torch.from_numpy(xs).cuda()
        samp = synth.density_sample(n_shard, cfg="C5")
        codes, quant = aqr.encode(x, sample_idx=torch.from_numpy(samp).cuda(), p_max=P_MAX["C5"], want_rho=True)
        torch.cuda.synchronize()
        eta = G.eta_of(G.density_weights(xs[samp], quant.rho.cpu().numpy(), literal=WJ_LITERAL))
        M, efc = G.adapt_params(32, 200, quant.delta, eta)
        lu = synth.level_draws(n_shard, cfg="C5", shard=s_)
        if BUILDER == "gpu":
            g = G.build_hnsw_gpu(codes, 96, M, efc, lu, flags=BUILD_FLAGS)
        else:
            g = G.build_hnsw(codes.cpu().numpy(), M, efc, lu, threads, flags=BUILD_FLAGS)
        ix = aqr.upload_index(codes, x, quant, g, metric="l2", id_base=s_ * n_shard, layout=LAYOUT)
        shards.append((x, ix, aqr.Searcher(ix, nq, aqr.make_params(k, **m, visited_bits=args.vbits[0]))))
        # exact ground truth of this shard (global ids), merged across shards below
        gi, gd = E.ground_truth(x, q, k)
        gt_i_parts.append(gi + s_ * n_shard)
        gt_d_parts.append(gd)
        infos.append(dict(shard=s_, M=M, efc=efc, delta=quant.delta, eta=eta, max_level=g.max_level,
                          build_s=round(time.time() - t0, 1), index_bytes=ix.device_bytes()))
        if rank == 0:
            log(f"[bench] C5 shard {s_}: {infos[-1]}")
        if rank == 0 and s_ == 0 and not (args.no_cpu or args.no_oracle):
            keep0 = (xs, samp, codes, g)  # shard 0's inputs for the cpu_baseline leg

    # the shards of a rank are searched concurrently on their own streams, so the persistent
    # grids of consecutive shards overlap instead of each launch paying its own tail
    side = [torch.cuda.Stream() for _ in shards] if args.shard_streams and len(shards) > 1 else None

    # --exchange peer: no NCCL on the data path.  Rank r owns query block r; every (shard, owner)
    # search writes its top-k straight into the owner's gather buffer (peer-mapped over NVLink),
    # then signal / wait / one merge of all S lists of the own block (parallel.PeerExchange)
    ex = None
    if args.exchange == "peer":
        ex = P.PeerExchange(aqr, nq, k, S)
        blocks = [P.block_range(nq, world, o)[:2] for o in range(world)]
        pstreams = [torch.cuda.Stream() for _ in range(min(8, len(shards) * world))]
        psearch = [[aqr.Searcher(sh[1], max(ex.blk, 1), aqr.make_params(k, **m, visited_bits=args.vbits[0]))
                    for _ in range(world)] for sh in shards]

    def step_peer():
        _, par = ex.begin()
        main = torch.cuda.current_stream()
        ready = torch.cuda.Event()
        ready.record(main)
        for st in pstreams:
            st.wait_event(ready)
        j = 0
        for si, s_ in enumerate(mine):
            for o, (lo, hi) in enumerate(blocks):
                if hi > lo:
                    psearch[si][o].run(q[lo:hi], stream=pstreams[j % len(pstreams)], out=ex.dest(o, s_, par))
                    j += 1
        for st in pstreams:
            main.wait_stream(st)
        ld, li = ex.finish(main)
        md, mi = aqr.merge_topk(ld, li)
        return md[: ex.hi - ex.lo], mi[: ex.hi - ex.lo]

    def step():
        if ex is not None:
            return step_peer()
        if side is None:
            outs = [sh[2].run(q) for sh in shards]
        else:
            main = torch.cuda.current_stream()
            ready = torch.cuda.Event()
            ready.record(main)
            outs = []
            for sh, st in zip(shards, side):
                st.wait_event(ready)
                outs.append(sh[2].run(q, stream=st))
            for st in side:
                main.wait_stream(st)
        if len(outs) == 1:
            ld, li = outs[0][1], outs[0][0]
        else:
            ld, li = aqr.merge_topk(torch.stack([o[1] for o in outs]), torch.stack([o[0] for o in outs]))
        return P.gather_merge(ld, li, aqr.merge_topk)

    # recall@10 / @100 against the merged exact ground truth (C5 is continuous: no exact ties)
    fd, fi = step()
    torch.cuda.synchronize()
    if ex is not None:
        ex.check()
        fd, fi = P.gather_rows(fd), P.gather_rows(fi)  # reporting only: every rank's merged block
        if args.check_exchange:
            # the NCCL path on the same inputs must give the same lists
            ex_keep, ex = ex, None
            rd, ri = step()
            ex = ex_keep
            torch.cuda.synchronize()
            same = bool(torch.equal(ri, fi) and torch.equal(rd, fd))
            log(f"[bench] rank {rank}: peer exchange == NCCL all-gather + merge: {same}")
            assert same, "peer exchange result differs from the NCCL path"
    gd_all = np.concatenate(gt_d_parts, 1)
    gi_all = np.concatenate(gt_i_parts, 1)
    if world > 1:
        td, ti = P.all_gather_lists(torch.from_numpy(gd_all).cuda(), torch.from_numpy(gi_all).cuda())
        gd_all = np.concatenate(list(td.cpu().numpy()), 1)
        gi_all = np.concatenate(list(ti.cpu().numpy()), 1)
    order = np.lexsort((gi_all, gd_all), axis=1)[:, :k]
    gt_ids = np.take_along_axis(gi_all, order, 1)
    found = fi.cpu().numpy()
    r10 = E.recall(found, gt_ids, k=10)[0]
    r100 = E.recall(found, gt_ids, k=100)[0]

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    clocks = Clocks(local)
    clocks.start()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    ms = allreduce_max(e0.elapsed_time(e1) / args.steps, world)
    value = nq / (ms / 1e3)
    # search-kernel share + counters (one untimed stats pass)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for sh in shards:
        sh[2].run(q)
    k1.record(stream)
    torch.cuda.synchronize()
    kern_ms = k0.elapsed_time(k1)
    bq_tot = 0.0
    ratios = []
    for sh in shards:
        # distinct-evaluation ratio of the shard, measured on the GPU: with the exact visited bitmap
        # (visited_bits -2) the kernel's evaluation count IS the oracle's distinct count
        # (tests/test_gpu_visited.py), so evals(-2) / evals(default) converts the default count
        ev = []
        for vb in (-2, args.vbits[0]):
            ss = aqr.Searcher(sh[1], nq, aqr.make_params(k, **m, visited_bits=vb))
            ss.totals.zero_()
            ss.run(q, stats=True)
            torch.cuda.synchronize()
            ev.append(ss.totals.cpu().numpy())
        ratio_s = float(ev[0][2]) / max(float(ev[1][2]), 1.0)
        ratios.append(round(ratio_s, 4))
        bq_tot += bytes_per_query(ev[1], nq, 96, k, ratio_s)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bq_tot * nq / (kern_ms / 1e3) / 1e9
    # end to end: pinned host queries in, host top-k out
    qh = torch.from_numpy(q_host).pin_memory()
    ids_h = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    dist_h = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    barrier(world)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(args.steps):
        q.copy_(qh, non_blocking=True)  # step() searches q
        rd, ri = step()  # peer exchange: this rank's merged block; NCCL path: all nq rows
        ids_h[: ri.shape[0]].copy_(ri, non_blocking=True)
        dist_h[: rd.shape[0]].copy_(rd, non_blocking=True)
    a1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = allreduce_max(a0.elapsed_time(a1) / args.steps, world)
    cpu = None
    if rank == 0 and keep0 is not None:
        cpu = cpu_baseline_sharded(keep0, q_host, shards[0][2], m, k, S, args.cpu_seconds)
        log(f"[bench] C5 cpu_baseline {cpu}")
    if rank == 0:
        line = {
            "metric": "QPS (C5 sharded, recall@10 reported)", "value": round(value, 1), "unit": "queries/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8+int32+f32",
            "data": "synthetic (seeded, BASELINE.json configs[4] recipe)",
            "config": {"workload": f"C5: {S} shards x {n_shard} x 96 l2, {nq} queries, k={k}", "ef": m["ef"],
                       "n_coarse": m["n_coarse"], "n_rerank": m["n_rerank"], "recall@10": round(r10, 4),
                       "recall@100": round(r100, 4),
                       "parallelism": (f"{S} shards over {world} GPU(s), NCCL all-gather + merge" if ex is None else
                                       f"{S} shards over {world} GPU(s), peer-memory exchange (search epilogue stores "
                                       f"into the block owner's buffer, signal/wait, one merge per block; no NCCL)"),
                       "exchange": args.exchange,
                       "shards_per_rank": len(mine), "visited_bits": args.vbits[0],
                       "warps_per_query": aqr.search_plan(shards[0][1], nq, shards[0][2].params) if shards else None,
                       "l2": "shard indexes > 126 MB L2; no flush", "shards": infos},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": None, "bytes_per_query": round(bq_tot, 1),
                         "kernel": "search_kernel (all shards of rank 0)", "kernel_ms": round(kern_ms, 4),
                         "distinct_eval_ratio_per_shard": ratios,
                         "note": "bytes from kernel counters; distinct evaluations per shard measured with the exact "
                                 "visited bitmap (equal to the oracle's distinct count, test_gpu_visited)"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(nq / (e2e_ms / 1e3), 1), "unit": "queries/s", "h2d_bytes_per_step": int(q_host.nbytes),
                    "d2h_bytes_per_step": int(nq * k * 8)},
            "gpu_launches": args.steps * ((len(shards) + (1 if len(shards) > 1 else 0) + (1 if world > 1 else 0)) if ex is None
                                          else (len(shards) * sum(1 for lo_, hi_ in blocks if hi_ > lo_) + 3)),
            "lib": aqr.lib().aqr_version().decode(),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if ex is not None:
        torch.cuda.synchronize()
        ex.check()
        ex.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# --------------------------------------------------------------------------------------------
# the reference arm: the CPU oracle as it stands (this tier has no reference implementation)
# --------------------------------------------------------------------------------------------
def mode_mapping(ef_mapping, ef, k, mode, sq8=False):
    """Search parameters of a re-rank mapping at ef (both arms; `ef_mapping` is the binding's or the
    oracle's copy of DESIGN.md R13).  "preset": Table 3 "0.97+" (R13); "full": the same N_c with every C
    entry re-ranked exactly (N_rerank = N_c) -- the Fig. 3 knob for data where d^q / d^a order is noisy
    (R20); "exact": full with the early-termination thresholds at infinity (R26), so a d^a gap can
    no longer cut the exact re-rank to k.  "<mode>/<m>": the same with the EF multiplier m_ef = m
    (ef_search = N_c x m_ef; Table 3 recommends 2-3; R29)."""
    mode, _, mef = mode.partition("/")
    mm = ef_mapping(ef, k, m_ef=int(mef) if mef else 3)
    if mode in ("full", "exact") or sq8:
        mm["n_rerank"] = mm["n_coarse"]
    if mode == "exact" or sq8:  # sq8: plain SQ8 HNSW (R23), every C entry re-ranked exactly
        mm["early_term"] = False
    return mm


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import synth
    from paper_2602_21600_b200 import graph as G
    cfg = args.config
    w = make_workload(cfg, args.scale, args.nq)
    k = w.k
    sample = synth.density_sample(len(w.x), seed=w.seed, cfg=cfg)
    t0 = time.time()
    rho = oracle.density(w.x, sample)
    delta = oracle.delta(rho)
    quant = oracle.train(w.x, sample, p_max=P_MAX[cfg], delta_override=delta)
    codes = oracle.encode(w.x, quant)
    eta = G.eta_of(G.density_weights(w.x[sample], rho, literal=WJ_LITERAL))
    M, efc = G.adapt_params(w.M0, w.efc0, quant.delta, eta)
    g = G.build_hnsw(codes, M, efc, synth.level_draws(len(w.x), seed=w.seed, cfg=cfg), args.threads,
                     flags=BUILD_FLAGS)
    log(f"[reference] index built in {time.time() - t0:.1f} s")
    ef, mode = AT_TARGET.get(cfg, (256, "preset"))
    if args.ef != "auto":
        ef = int(args.ef)
    if args.rerank not in ("auto", None) and "," not in args.rerank:
        mode = args.rerank
    m = mode_mapping(oracle.ef_mapping, ef, k, mode)
    oix = oracle.Index(w.x, codes, quant, g, w.metric)
    cores = os.cpu_count() or 1
    t0 = time.time()
    oracle.search(oix, w.q[:4], k, **m)
    per_q = max((time.time() - t0) / 4, 1e-6)
    per_step = int(max(cores, min(len(w.q), cores * args.cpu_seconds / max(1, args.steps + args.warmup) / per_q)))
    for _ in range(args.warmup):
        oracle_search_threads(oix, w.q[:per_step], k, cores, **m)
    t0 = time.time()
    for _ in range(args.steps):
        oracle_search_threads(oix, w.q[:per_step], k, cores, **m)
    el = time.time() - t0
    v = per_step * args.steps / el
    line = {"impl": "reference", "metric": "QPS at recall@10>=0.98", "value": round(v, 2), "unit": "queries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(el / args.steps * 1e3, 2), "higher_is_better": True,
            "scaling": "strong" if cfg == "C5" else args.scaling,
            "vs_baseline": None, "dtype": "u8+int32+f32", "data": "synthetic",
            "config": {"workload": f"{cfg}: {len(w.x)} x {w.x.shape[1]} {w.metric}, {len(w.q)} queries, k={k}",
                       "rerank": mode, **m},
            "cpu_baseline": {"value": round(v, 2), "unit": "queries/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"{per_step} queries per step (a bounded sample of the config's set), the "
                                       f"single-threaded C oracle run query-parallel on {cores} host threads"},
            "e2e": {"value": round(v, 2), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="aqr", choices=["aqr", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of the config's base size")
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--ef", default="auto")
    ap.add_argument("--full-sweep", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="C5: how the per-shard top-k lists meet -- nccl: all_gather_into_tensor + merge (default); "
                         "peer: aqr_search stores into the block owner's peer-mapped buffer, aqr_peer_signal / "
                         "aqr_peer_wait, one merge per block (no NCCL on the data path)")
    ap.add_argument("--check-exchange", action="store_true", help="C5 --exchange peer: assert the NCCL path gives the same lists")
    ap.add_argument("--shard-streams", type=int, default=1,
                    help="C5: search a rank's shards concurrently on separate CUDA streams (1) or one after another (0)")
    ap.add_argument("--stream", type=int, default=0,
                    help="also time a steady-state stream of this many fresh queries (C1/C4 under-fill the GPU)")
    ap.add_argument("--traversal", default="aqr", choices=["aqr", "fp32", "sq8"],
                    help="aqr: the method; fp32: the paper's baseline HNSW search on the same graph; sq8: the "
                         "paper's plain scalar-quantization HNSW (delta = 0 codes and graph, no early termination, "
                         "full exact re-rank; R23) (NEXT-2)")
    ap.add_argument("--rerank", default="auto",
                    help="re-rank mappings swept: preset (Table 3, N_rerank = 28), full (N_rerank = N_c), exact (full, "
                         "early termination off); auto = preset for C2 (identical recall there, measured), all three "
                         "otherwise")
    ap.add_argument("--vbits", type=lambda v: [int(t) for t in v.split(",")], default=None,
                    help="visited sets tried at the chosen ef, fastest is timed (write --vbits=-1,12): -1 none, "
                         "6..16 a shared-memory hash of 2^v slots, -2 the exact global bitmap.  Default: -2,-1,13 "
                         "for C1, -2,-1 for C4 (re-evaluations dominate there), -1 otherwise (R15)")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-oracle", action="store_true", help="skip the oracle index (no cpu_baseline, ratio 1)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="C1-C4 over N GPUs: weak = N x nq distinct queries, nq per rank (default); strong = "
                         "the config's nq split across the ranks")
    ap.add_argument("--layout", default="auto", choices=["auto", "gather", "inline"])
    ap.add_argument("--tau-spread", type=float, default=float("inf"),
                    help="adaptive re-rank depth (P:154, R27): re-rank only the entries of A within (1 + tau) of "
                         "d^a_k (at least k, at most N_rerank); inf = the static N_rerank (default)")
    ap.add_argument("--pipeline", type=int, default=2,
                    help="C1-C4: streams the timed steps are issued on, round-robin (1 = back to back on one "
                         "stream); each stream has its own Searcher, so a step's tail overlaps the next step")
    ap.add_argument("--builder", default="gpu", choices=["gpu", "host"],
                    help="graph construction (not timed): gpu = aqr_build_graph (NEXT-1), host = csrc/hnsw_build.cpp; "
                         "both give the same graph byte for byte")
    ap.add_argument("--wj", default="spec", choices=["spec", "literal"],
                    help="density weights w_j for eta (builder only): spec = SPEC's per-dimension weighted "
                         "variance (R16, default); literal = Alg1 l.12 as printed (eta = 0)")
    args = ap.parse_args()
    global LAYOUT, WJ_LITERAL, BUILDER
    WJ_LITERAL = args.wj == "literal"
    BUILDER = args.builder
    LAYOUT = args.layout
    if args.warmup < 3:
        log("[bench] warm-up raised to 3 (timing rule)")
        args.warmup = 3
    args.kt = "fp32" if args.traversal == "fp32" else "aqr"  # the kernel's traversal
    if args.vbits is None:
        # the exact global visited bitmap (-2) pays where re-evaluations dominate (distinct ratio
        # 0.03 on C1, 0.09 on C4: measured 2.2x / 3.3x); C5 (0.09 per shard) a 2^10-slot 16-bit-tag
        # table in shared memory (no occupancy cost: 3.79 -> 2.97 ms per shard); elsewhere none (R15)
        args.vbits = {"C1": [-2, -1, 13], "C4": [-2, -1], "C5": [10]}.get(args.config, [-1])
    if args.traversal == "sq8":
        args.rerank = "full"
    if args.rerank == "auto":
        args.rerank = "preset" if args.config == "C2" else "preset,full,exact"
    if args.impl != "reference":
        rc = relaunch_if_needed(args)
        if rc is not None:
            sys.exit(rc)
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "C5":
        run_sharded(args)
    else:
        run_aqr(args)


if __name__ == "__main__":
    main()
