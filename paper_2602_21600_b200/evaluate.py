"""Evaluation helpers (not the search path): exact ground truth and recall@k.

Ground truth: brute force on the GPU with torch (fp32 matmul with TF32 off for a shortlist of
k + 32 candidates per query, re-scored in fp64, ties broken by id).  Recall@k ("the
fraction of true top-10 neighbours retrieved"): the id overlap with the ground truth, plus
the tie-aware variant used by ann-benchmarks (a returned id counts when its exact distance is
<= the true k-th distance), which is the headline number because integer data (C2) has exact
distance ties at the k-th position (R18)."""
from __future__ import annotations

import numpy as np
import torch


@torch.no_grad()
def ground_truth(x: torch.Tensor, q: torch.Tensor, k: int, metric: str = "l2", extra: int = 32,
                 chunk: int = 1 << 18):
    """Exact top-k ids [nq, k] int64 and fp64 distances (L2 squared, or 1 - <q,x> for IP)."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        kk = min(k + extra, x.shape[0])
        qn = (q.double() ** 2).sum(1).float()
        best_d = None
        best_i = None
        for s in range(0, x.shape[0], chunk):
            xs = x[s:s + chunk]
            if metric == "l2":
                d = qn[:, None] + (xs.double() ** 2).sum(1).float()[None, :] - 2.0 * (q @ xs.T)
            else:
                d = 1.0 - q @ xs.T
            kc = min(kk, d.shape[1])
            v, i = torch.topk(d, kc, dim=1, largest=False)
            i = i + s
            if best_d is None:
                best_d, best_i = v, i
            else:
                cat_d = torch.cat([best_d, v], 1)
                cat_i = torch.cat([best_i, i], 1)
                v2, o = torch.topk(cat_d, min(kk, cat_d.shape[1]), dim=1, largest=False)
                best_d, best_i = v2, torch.gather(cat_i, 1, o)
        ed = exact_dist(x, q, best_i, metric)
        # sort by (fp64 distance, id)
        order = np.lexsort((best_i.cpu().numpy(), ed.cpu().numpy()), axis=1)
        ids = np.take_along_axis(best_i.cpu().numpy(), order, 1)[:, :k]
        dd = np.take_along_axis(ed.cpu().numpy(), order, 1)[:, :k]
        return ids, dd
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


@torch.no_grad()
def exact_dist(x: torch.Tensor, q: torch.Tensor, ids: torch.Tensor, metric: str = "l2", chunk: int = 2048):
    """fp64 exact distances of q[i] to x[ids[i, j]]; ids < 0 give +inf."""
    out = torch.empty(ids.shape, dtype=torch.float64, device=x.device)
    for s in range(0, ids.shape[0], chunk):
        ii = ids[s:s + chunk].long()
        valid = ii >= 0
        xv = x[ii.clamp_min(0)].double()
        qv = q[s:s + chunk].double()[:, None, :]
        if metric == "l2":
            d = ((xv - qv) ** 2).sum(-1)
        else:
            d = 1.0 - (xv * qv).sum(-1)
        out[s:s + chunk] = torch.where(valid, d, torch.full_like(d, float("inf")))
    return out


def recall(found_ids: np.ndarray, gt_ids: np.ndarray, found_exact_d: np.ndarray | None = None,
           gt_d: np.ndarray | None = None, k: int = 10, rel: float = 1e-6):
    """(id-overlap recall, tie-aware recall) averaged over queries."""
    f = found_ids[:, :k]
    g = gt_ids[:, :k]
    overlap = np.mean([len(set(a[a >= 0].tolist()) & set(b.tolist())) / k for a, b in zip(f, g)])
    if found_exact_d is None or gt_d is None:
        return float(overlap), float(overlap)
    thr = gt_d[:, k - 1:k]
    tol = rel * np.maximum(np.abs(thr), 1.0)
    hits = np.minimum((found_exact_d[:, :k] <= thr + tol).sum(1), k)
    return float(overlap), float(np.mean(hits / k))
