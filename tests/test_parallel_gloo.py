"""N > 1 host path on CPU: world_size-2 gloo process groups.

The sharded (C5) path gathers every rank's per-shard-merged top-k lists and merges them again;
the result must be byte-identical to one merge over all shards (the merge orders by
(dist, global id), BASELINE.json configs[4]).  The merge used here is the oracle's
(oracle.merge_topk); on the GPU the same plumbing calls aqr.merge_topk."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2602_21600_b200 import parallel as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_lists(S, nq, k, seed=5):
    """Per-shard sorted (dist, global id) lists with many exact distance ties and short lists."""
    rng = np.random.default_rng(seed)
    d = rng.integers(0, 30, size=(S, nq, k)).astype(np.float32) / 8
    ids = np.stack([rng.permutation(5000)[: nq * k].reshape(nq, k) + s * 5000 for s in range(S)]).astype(np.int32)
    order = np.lexsort((ids, d), axis=-1)
    d = np.take_along_axis(d, order, -1)
    ids = np.take_along_axis(ids, order, -1)
    d[1, 3, -4:] = np.inf  # a short shard list (padded with (-1, +inf))
    ids[1, 3, -4:] = -1
    return d, ids


def _merge(od, oi):
    k = od.shape[-1]
    md, mi = oracle.merge_topk(od.numpy(), oi.numpy(), k)
    return torch.from_numpy(md), torch.from_numpy(mi)


def _worker(rank, world, port, S, nq, k, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, ids = _shard_lists(S, nq, k)
        mine = P.shards_of_rank(S, world, rank)
        # local merge over this rank's shards, then the cross-rank gather + merge
        ld, li = _merge(torch.from_numpy(d[mine]), torch.from_numpy(ids[mine]))
        gd, gi = P.gather_merge(ld, li, _merge)
        # replicated path: each rank's query slice, gathered back in rank order
        lo, hi = P.query_range(nq, world, rank)
        rows = P.gather_rows(torch.arange(lo, hi, dtype=torch.int64))
        np.save(os.path.join(out_dir, f"r{rank}_d.npy"), gd.numpy())
        np.save(os.path.join(out_dir, f"r{rank}_i.npy"), gi.numpy())
        np.save(os.path.join(out_dir, f"r{rank}_rows.npy"), rows.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_gather_merge_gloo(tmp_path, world):
    S, nq, k = 8, 37, 12
    mp.spawn(_worker, args=(world, _free_port(), S, nq, k, str(tmp_path)), nprocs=world, join=True)
    d, ids = _shard_lists(S, nq, k)
    ref_d, ref_i = oracle.merge_topk(d, ids, k)
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"r{r}_i.npy"), ref_i)
        np.testing.assert_array_equal(np.load(tmp_path / f"r{r}_d.npy").view(np.uint32), ref_d.view(np.uint32))
        np.testing.assert_array_equal(np.load(tmp_path / f"r{r}_rows.npy"), np.arange(nq))


def test_partitions():
    for nq in [0, 1, 7, 10_000]:
        for world in [1, 2, 3, 8]:
            spans = [P.query_range(nq, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nq
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    for world in [1, 2, 4, 8]:
        got = sorted(s for r in range(world) for s in P.shards_of_rank(8, world, r))
        assert got == list(range(8))
    assert [P.shard_rows(10_000_000, 8, s) for s in (0, 7)] == [(0, 1_250_000), (8_750_000, 10_000_000)]
    with pytest.raises(ValueError):
        P.shards_of_rank(8, 3, 0)


def test_single_process_without_group():
    """A single-GPU run never initialises a process group: the plumbing is the identity."""
    assert not dist.is_initialized()
    d = torch.arange(6, dtype=torch.float32).reshape(2, 3)
    i = torch.arange(6, dtype=torch.int32).reshape(2, 3)
    gd, gi = P.gather_merge(d, i, _merge)
    assert gd is d and gi is i
    assert P.gather_rows(i) is i
    od, oi = P.all_gather_lists(d, i)
    assert od.shape == (1, 2, 3) and oi.shape == (1, 2, 3)


def _weak_worker(rank, world, port, cfg, nq, out_dir):
    """The replicated-index weak-scaling split of bench.py: each rank materialises its own query
    block (P.weak_block) and the blocks are gathered back in rank order."""
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        src, lo, hi = P.weak_block(nq, world, rank)
        if src == "config":
            q = synth.gen_config(cfg, scale=0.001, nq=nq).q
        else:
            q = synth.gen_query_stream(cfg, hi)[lo:hi]
        allq = P.gather_rows(torch.from_numpy(np.ascontiguousarray(q)))
        np.save(os.path.join(out_dir, f"w{rank}.npy"), allq.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_weak_scaling_queries_are_distinct_gloo(tmp_path, world):
    """bench.py C1-C4 over N ranks (default weak scaling): N x nq DISTINCT queries, nq per rank --
    rank 0 the config's query set, rank r >= 1 rows [(r-1) nq, r nq) of synth stream 3 -- never
    the same queries counted once per GPU."""
    import synth
    cfg, nq = "C2", 50
    mp.spawn(_weak_worker, args=(world, _free_port(), cfg, nq, str(tmp_path)), nprocs=world, join=True)
    want = np.concatenate([synth.gen_config(cfg, scale=0.001, nq=nq).q,
                           synth.gen_query_stream(cfg, (world - 1) * nq)])
    for r in range(world):
        got = np.load(tmp_path / f"w{r}.npy")
        np.testing.assert_array_equal(got, want)
    assert len(np.unique(want, axis=0)) == world * nq


def test_weak_blocks():
    for world in [1, 2, 8]:
        blocks = [P.weak_block(10_000, world, r) for r in range(world)]
        assert blocks[0] == ("config", 0, 10_000)
        assert [b[1:] for b in blocks[1:]] == [((r - 1) * 10_000, r * 10_000) for r in range(1, world)]


def test_bench_refuses_world_mismatch(monkeypatch):
    """--gpus N must equal WORLD_SIZE under torchrun; without torchrun, N > 1 relaunches."""
    import argparse
    import bench
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.relaunch_if_needed(argparse.Namespace(gpus=4)) == 2
    assert bench.relaunch_if_needed(argparse.Namespace(gpus=2)) is None
    monkeypatch.delenv("WORLD_SIZE")
    assert bench.relaunch_if_needed(argparse.Namespace(gpus=1)) is None
