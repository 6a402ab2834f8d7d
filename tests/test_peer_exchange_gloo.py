"""parallel.PeerExchange on CPU (world_size-2 and -3 gloo groups): the host logic of the C5
peer-memory exchange -- layout, handle exchange, destination addresses, step / parity, signal and
wait -- driven through a stand-in for the binding's peer_* calls that uses POSIX shared memory
between the rank processes (on the GPU the same calls are aqr_peer_alloc / aqr_peer_open over
CUDA IPC and the signal / wait kernels).  Each "search" writes its shard's top-k rows of one
query block straight into the block owner's buffer, as aqr_search does with a peer-mapped
out pointer.  The merged blocks must equal one merge over all shards (oracle.merge_topk)."""
import ctypes
import os
import socket
import time
from multiprocessing import shared_memory

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2602_21600_b200 import parallel as P


def _shard_lists(S, nq, k, seed=5):
    """Per-shard sorted (dist, global id) lists with many exact distance ties."""
    rng = np.random.default_rng(seed)
    d = rng.integers(0, 30, size=(S, nq, k)).astype(np.float32) / 8
    ids = np.stack([rng.permutation(5000)[: nq * k].reshape(nq, k) + s * 5000 for s in range(S)]).astype(np.int32)
    order = np.lexsort((ids, d), axis=-1)
    d = np.take_along_axis(d, order, -1)
    ids = np.take_along_axis(ids, order, -1)
    if S > 1 and nq > 3:
        d[1, 3, -4:] = np.inf  # a short shard list (padded with (-1, +inf))
        ids[1, 3, -4:] = -1
    return d, ids


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _Buf:
    def __init__(self, shm, owner):
        self.shm, self.owner = shm, owner
        self.nbytes = shm.size
        self._c = (ctypes.c_uint8 * shm.size).from_buffer(shm.buf)
        self.ptr = ctypes.addressof(self._c)
        self.handle = shm.name.encode().ljust(64, b"\0")

    def tensor(self, dtype, shape, offset=0):
        n = int(np.prod(shape))
        return torch.frombuffer(self.shm.buf, dtype=dtype, count=n, offset=offset).view(*shape)

    def close(self):
        del self._c
        try:
            self.shm.close()
            if self.owner:
                self.shm.unlink()
        except BufferError:
            pass


class FakeAqr:
    """The binding's peer_* surface over shared memory (addresses are this process's mappings)."""
    MAX_PEERS = 8

    @staticmethod
    def peer_alloc(nbytes):
        shm = shared_memory.SharedMemory(create=True, size=nbytes)
        shm.buf[:nbytes] = bytes(nbytes)
        return _Buf(shm, True)

    @staticmethod
    def peer_open(handle, nbytes):
        return _Buf(shared_memory.SharedMemory(name=handle.rstrip(b"\0").decode()), False)

    @staticmethod
    def peer_signal(flag_ptrs, slot, value, stream=None):
        for p in flag_ptrs:
            ctypes.c_uint64.from_address(p + 8 * slot).value = value

    @staticmethod
    def peer_wait(flags_ptr, n, value, timeout_ns, status=None, stream=None):
        t0 = time.time()
        for i in range(n):
            while ctypes.c_uint64.from_address(flags_ptr + 8 * i).value < value:
                if (time.time() - t0) * 1e9 > timeout_ns:
                    status[0] = 1 + i
                    return
                time.sleep(0.0005)


def _put(ptr, arr):
    a = np.ascontiguousarray(arr)
    ctypes.memmove(ptr, a.ctypes.data, a.nbytes)


def _worker(rank, world, port, S, nq, k, steps, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = None
    try:
        ex = P.PeerExchange(FakeAqr, nq, k, S, timeout_s=20.0, device="cpu")
        mine = P.shards_of_rank(S, world, rank)
        for step in range(steps):
            d, ids = _shard_lists(S, nq, k, seed=5 + step)  # fresh lists every step (parity reuse)
            _, par = ex.begin()
            for s_ in mine:  # the "search" of shard s_ on query block o lands in rank o's buffer
                for o in range(world):
                    lo, hi, _ = P.block_range(nq, world, o)
                    if hi > lo:
                        p_ids, p_dist = ex.dest(o, s_, par)
                        _put(p_ids, ids[s_, lo:hi])
                        _put(p_dist, d[s_, lo:hi])
            ld, li = ex.finish()
            ex.check()
            n_b = ex.hi - ex.lo
            md, mi = oracle.merge_topk(ld[:, :n_b].numpy().copy(), li[:, :n_b].numpy().copy(), k)
            np.save(os.path.join(out_dir, f"s{step}_r{rank}_d.npy"), md)
            np.save(os.path.join(out_dir, f"s{step}_r{rank}_i.npy"), mi)
        del ld, li
    finally:
        if ex is not None:
            ex.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,S,nq", [(2, 8, 37), (3, 3, 10), (2, 2, 1)])
def test_peer_exchange_equals_one_merge(tmp_path, world, S, nq):
    k, steps = 12, 3
    mp.spawn(_worker, args=(world, _free_port(), S, nq, k, steps, str(tmp_path)), nprocs=world, join=True)
    for step in range(steps):
        d, ids = _shard_lists(S, nq, k, seed=5 + step)
        ref_d, ref_i = oracle.merge_topk(d, ids, k)
        got_i = np.concatenate([np.load(tmp_path / f"s{step}_r{r}_i.npy") for r in range(world)])
        got_d = np.concatenate([np.load(tmp_path / f"s{step}_r{r}_d.npy") for r in range(world)])
        np.testing.assert_array_equal(got_i, ref_i)
        np.testing.assert_array_equal(got_d.view(np.uint32), ref_d.view(np.uint32))


def test_block_range_and_layout():
    for nq in [0, 1, 7, 37, 10_000]:
        for world in [1, 2, 3, 8]:
            spans = [P.block_range(nq, world, o) for o in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nq
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(hi - lo <= blk for lo, hi, blk in spans) and len({b for _, _, b in spans}) == 1
    lay = P.exchange_layout(8, 1250, 100, 8)
    regions = sorted([(lay["ids"][0], lay["list_bytes"]), (lay["dist"][0], lay["list_bytes"]),
                      (lay["ids"][1], lay["list_bytes"]), (lay["dist"][1], lay["list_bytes"]), (lay["flags"], 64)])
    assert all(a[0] + a[1] <= b[0] for a, b in zip(regions, regions[1:]))  # disjoint
    assert regions[-1][0] + regions[-1][1] <= lay["total"] and lay["list_bytes"] >= 8 * 1250 * 100 * 4
    assert all(off % 256 == 0 for off, _ in regions)
    with pytest.raises(ValueError):
        P.exchange_layout(33, 10, 10, 2)


def test_wait_times_out_when_a_rank_never_signals():
    ex = P.PeerExchange(FakeAqr, 4, 2, 1, timeout_s=0.05, device="cpu")
    try:
        ex.world = 2  # pretend a second rank exists that never signals
        ex.begin()
        FakeAqr.peer_signal([ex.local.ptr + ex.lay["flags"]], 0, ex.step)
        FakeAqr.peer_wait(ex.local.ptr + ex.lay["flags"], 2, ex.step, ex.timeout_ns, ex.status)
        with pytest.raises(RuntimeError, match="rank 1"):
            ex.check()
    finally:
        ex.world = 1
        ex.close()
