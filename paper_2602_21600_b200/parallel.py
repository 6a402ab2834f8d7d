"""Multi-GPU plumbing of the batched search: one process per GPU, torch.distributed.

* C1-C4 -- replicas.  Every rank holds the whole index and searches distinct queries: for weak
  scaling (the default) each rank its own block of nq (`weak_block`, world x nq queries in all),
  for strong scaling a contiguous slice of one batch (`query_range`).  No collective on the data
  path; `gather_rows` collects per-rank result rows for reporting only.
* C5 -- the base is sharded S ways (BASELINE.json configs[4]); rank r holds the shards
  `shards_of_rank(S, world, r)`, each a complete AQR index whose ids are offset by the shard's
  first row (`shard_rows`, passed to aqr_upload_index as id_base).  Per rank the per-shard top-k
  lists are merged by aqr_merge_topk, the per-rank lists are gathered over NCCL
  (`all_gather_into_tensor` of [nq x k] dists + ids, NVLink / NVSwitch) and merged again
  (`gather_merge`).  The merge orders by (dist, global id), so the output is
  identical for every world size.

* C5 over peer memory (`PeerExchange`, opt-in: `bench.py --exchange peer`): no NCCL call on the
  data path.  Rank r owns query block r (`block_range`).  Every rank searches each block on its
  shard(s) with aqr_search writing straight into the owner's gather buffer (peer-mapped over
  NVLink: the search epilogue's stores are the transfer), signals the owners, and each owner waits
  for all ranks and merges the S lists of its block (aqr_merge_topk).  The (dist, global id)
  merge makes the result identical to the NCCL path's.

Only plumbing lives here: the merge itself is a callable (aqr.merge_topk on the GPU path; the
CPU tests pass the oracle's merge through gloo).
"""
from __future__ import annotations


def query_range(nq: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous query slice [lo, hi) of `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return rank * nq // world, (rank + 1) * nq // world


def weak_block(nq: int, world: int, rank: int) -> tuple[str, int, int]:
    """Weak scaling of the replicated configs (C1-C4): the job is world x nq DISTINCT queries,
    rank r searches its own block of nq.  Rank 0's block is the config's query set (so the
    single-GPU run is the config itself); rank r >= 1 takes rows [(r-1) nq, r nq) of the
    config's supplementary query stream (synth stream 3).  Returns (source, lo, hi) with source
    "config" or "stream"."""
    if world < 1 or not 0 <= rank < world or nq < 0:
        raise ValueError("bad world/rank/nq")
    if rank == 0:
        return "config", 0, nq
    return "stream", (rank - 1) * nq, rank * nq


def shard_rows(n_total: int, n_shards: int, s: int) -> tuple[int, int]:
    """Base rows [lo, hi) of shard s (C5: 8 shards of 1.25M rows; shard base = lo = id_base)."""
    if n_shards < 1 or not 0 <= s < n_shards:
        raise ValueError("bad shard")
    return s * n_total // n_shards, (s + 1) * n_total // n_shards


def shards_of_rank(n_shards: int, world: int, rank: int) -> list[int]:
    """Shards held by `rank`: a contiguous block of n_shards / world (world must divide n_shards
    or exceed it; with world > n_shards the extra ranks hold nothing)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if world <= n_shards:
        if n_shards % world:
            raise ValueError("world size must divide the shard count")
        per = n_shards // world
        return list(range(rank * per, (rank + 1) * per))
    return [rank] if rank < n_shards else []


def _dist():
    import torch.distributed as dist
    return dist


def _world(group=None) -> int:
    """World size, 1 when no process group is initialised (a single-GPU run)."""
    d = _dist()
    return d.get_world_size(group) if d.is_available() and d.is_initialized() else 1


def all_gather_lists(dist_t, ids_t, group=None):
    """[nq, k] dists (fp32) + ids (int32) of every rank -> [world, nq, k] each, rank order."""
    import torch
    d = _dist()
    world = _world(group)
    if world == 1:
        return dist_t.unsqueeze(0), ids_t.unsqueeze(0)
    nq, k = dist_t.shape
    od = torch.empty((world, nq, k), dtype=dist_t.dtype, device=dist_t.device)
    oi = torch.empty((world, nq, k), dtype=ids_t.dtype, device=ids_t.device)
    if d.get_backend(group) == "nccl":
        d.all_gather_into_tensor(od, dist_t.contiguous(), group=group)
        d.all_gather_into_tensor(oi, ids_t.contiguous(), group=group)
    else:  # gloo (CPU tests): list form
        d.all_gather(list(od.unbind(0)), dist_t.contiguous(), group=group)
        d.all_gather(list(oi.unbind(0)), ids_t.contiguous(), group=group)
    return od, oi


def gather_merge(dist_t, ids_t, merge_fn, group=None):
    """Merge this rank's [nq, k] top-k list with every other rank's: all-gather, then
    merge_fn([world, nq, k] dists, ids) -> ([nq, k], [nq, k]) on every rank."""
    od, oi = all_gather_lists(dist_t, ids_t, group)
    if od.shape[0] == 1:
        return dist_t, ids_t
    return merge_fn(od, oi)


def gather_rows(t, group=None):
    """Concatenate per-rank row blocks (possibly of different lengths) in rank order."""
    import torch
    d = _dist()
    world = _world(group)
    if world == 1:
        return t
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    d.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    mx = max(ns)
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    d.all_gather(outs, pad, group=group)
    return torch.cat([o[:m] for o, m in zip(outs, ns)])


def block_range(nq: int, world: int, owner: int) -> tuple[int, int, int]:
    """Query block [lo, hi) merged by rank `owner` and the block stride blk = ceil(nq / world)
    (every gather buffer holds blk rows per list; the last block may be shorter or empty)."""
    if world < 1 or not 0 <= owner < world or nq < 0:
        raise ValueError("bad world/owner/nq")
    blk = (nq + world - 1) // world
    lo = min(owner * blk, nq)
    return lo, min(lo + blk, nq), blk


def exchange_layout(n_lists: int, blk: int, k: int, world: int) -> dict:
    """Byte offsets inside one rank's exchange allocation: two parities (step & 1) of
    ids [n_lists x blk x k] int32 and dist [n_lists x blk x k] fp32, then world uint64 flags."""
    if n_lists < 1 or n_lists > 32 or blk < 0 or k < 1 or world < 1:
        raise ValueError("bad exchange shape")
    lst = (n_lists * max(blk, 1) * k * 4 + 255) // 256 * 256
    return {"list_bytes": lst, "ids": [0, 2 * lst], "dist": [lst, 3 * lst], "flags": 4 * lst,
            "total": 4 * lst + (8 * world + 255) // 256 * 256}


class PeerExchange:
    """The C5 gather over peer memory (include/aqr.h "Peer-memory exchange"): allocation and handle
    exchange (one all_gather_object at set-up, never on the data path), destination pointers for
    aqr_search, and the per-step signal / wait.  `aqr` is the binding module."""

    def __init__(self, aqr, nq: int, k: int, n_lists: int, group=None, timeout_s: float = 20.0, device="cuda"):
        import torch
        d = _dist()
        self.aqr, self.nq, self.k, self.n_lists, self.group = aqr, nq, k, n_lists, group
        self.world = _world(group)
        self.rank = d.get_rank(group) if self.world > 1 else 0
        if self.world > aqr.MAX_PEERS:
            raise ValueError(f"at most {aqr.MAX_PEERS} ranks")
        self.lo, self.hi, self.blk = block_range(nq, self.world, self.rank)
        self.lay = exchange_layout(n_lists, self.blk, k, self.world)
        self.timeout_ns = int(timeout_s * 1e9)
        self.local = aqr.peer_alloc(self.lay["total"])
        self.peers = [self.local]
        if self.world > 1:
            handles = [None] * self.world
            d.all_gather_object(handles, self.local.handle, group=group)
            self.peers = [self.local if r == self.rank else aqr.peer_open(handles[r], self.lay["total"])
                          for r in range(self.world)]
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.step = 0

    def dest(self, owner: int, slot: int, parity: int) -> tuple[int, int]:
        """Device addresses (ids, dist) of list `slot` of query block `owner`, in the owner's buffer."""
        if not (0 <= owner < self.world and 0 <= slot < self.n_lists and parity in (0, 1)):
            raise ValueError("bad destination")
        off = slot * self.blk * self.k * 4
        base = self.peers[owner].ptr
        return base + self.lay["ids"][parity] + off, base + self.lay["dist"][parity] + off

    def begin(self) -> tuple[int, int]:
        """Start a step: (step number >= 1, parity).  Two parities suffice: a rank can start step
        s + 2 only after every rank signalled step s + 1, i.e. after every rank merged step s."""
        self.step += 1
        return self.step, self.step & 1

    def finish(self, stream=None):
        """After this rank's searches of the step were launched on `stream` (or on streams it
        waits for): signal every owner, wait for every rank, return the local views
        (dist [n_lists, blk, k], ids [n_lists, blk, k]) of this step's parity."""
        import torch
        flags = [p.ptr + self.lay["flags"] for p in self.peers]
        self.aqr.peer_signal(flags, self.rank, self.step, stream)
        self.aqr.peer_wait(flags[self.rank], self.world, self.step, self.timeout_ns, self.status, stream)
        par = self.step & 1
        shape = (self.n_lists, max(self.blk, 1), self.k)
        return (self.local.tensor(torch.float32, shape, self.lay["dist"][par]),
                self.local.tensor(torch.int32, shape, self.lay["ids"][par]))

    def check(self):
        """After a synchronize: raise if a wait timed out (a rank never signalled)."""
        v = int(self.status.item())
        if v:
            raise RuntimeError(f"peer exchange: rank {v - 1} did not signal step {self.step} in time")

    def close(self):
        d = _dist()
        for r, p in enumerate(self.peers):
            if r != self.rank:
                p.close()
        if self.world > 1:
            d.barrier(group=self.group)  # every peer unmapped before the owner frees
        self.local.close()
