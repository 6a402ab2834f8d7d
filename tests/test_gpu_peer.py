"""The peer-memory exchange on one GPU (include/aqr.h "Peer-memory exchange"): the
C-ABI pieces (aqr_peer_alloc / signal / wait / free) and parallel.PeerExchange in its world-size-1
form, where the block owner is this process and every "peer" pointer is local -- the same
kernels and the same addressing as across GPUs, minus cudaIpcOpenMemHandle (a process must not
open its own handle).  aqr_search writes each (shard, block) top-k list straight into the
gather buffer; the merged result must equal the stacked-lists merge and the oracle's.  The
multi-rank host logic is covered on CPU by tests/test_peer_exchange_gloo.py."""
import numpy as np
import pytest

import oracle
import synth
from paper_2602_21600_b200 import graph as G
from paper_2602_21600_b200 import parallel as P

pytestmark = pytest.mark.gpu

S, N_SHARD, NQ, K = 3, 2500, 37, 20


def test_alloc_signal_wait_timeout():
    import torch
    import paper_2602_21600_b200 as aqr
    buf = aqr.peer_alloc(4096)
    try:
        assert len(buf.handle) == aqr.PEER_HANDLE_BYTES and buf.handle != bytes(64)
        flags = buf.tensor(torch.int64, (8,), 1024)
        assert int(flags.abs().sum()) == 0  # zero-filled
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        fp = buf.ptr + 1024
        aqr.peer_signal([fp], 0, 7)
        aqr.peer_signal([fp, fp], 2, 9)  # several destinations (here the same array)
        aqr.peer_wait(fp, 1, 7, 5_000_000_000, status)
        torch.cuda.synchronize()
        assert flags.tolist()[:3] == [7, 0, 9] and int(status.item()) == 0
        # slot 1 was never signalled: the wait gives up after its timeout and names it
        aqr.peer_wait(fp, 3, 1, 20_000_000, status)
        torch.cuda.synchronize()
        assert int(status.item()) == 2
        with pytest.raises(aqr.AqrError):
            aqr.peer_signal([fp] * 9, 0, 1)
        with pytest.raises(aqr.AqrError):
            aqr.peer_wait(fp, 33, 1, 1000, status)
        with pytest.raises(aqr.AqrError):
            buf.tensor(torch.int32, (2048,), 0)  # past the end
    finally:
        buf.close()


def test_exchange_world1_matches_merge_and_oracle():
    import torch
    import paper_2602_21600_b200 as aqr
    q = synth.gen_c5_queries(NQ)
    qt = torch.from_numpy(q).cuda()
    m = aqr.ef_mapping(64, K)
    ixs, o_lists, keep = [], [], []
    for s in range(S):
        x = synth.gen_c5_shard(s, N_SHARD)
        samp = synth.density_sample(N_SHARD, cfg="C5")
        oq = oracle.train(x, samp, p_max=5.0)
        oc = oracle.encode(x, oq)
        g = G.build_hnsw(oc, 12, 48, synth.level_draws(N_SHARD, cfg="C5", shard=s), 4, flags=1)
        base = P.shard_rows(S * N_SHARD, S, s)[0]
        xt = torch.from_numpy(x).cuda()
        codes, quant = aqr.encode(xt, sample_idx=torch.from_numpy(samp).cuda(), p_max=5.0)
        ixs.append(aqr.upload_index(codes, xt, quant, g, metric="l2", id_base=base))
        keep.append((xt, codes, quant))
        oi, od = oracle.search(oracle.Index(x, oc, oq, g, "l2"), q, K, **m)
        o_lists.append((od, np.where(oi >= 0, oi + base, -1).astype(np.int32)))
    od, oi = oracle.merge_topk(np.stack([d for d, _ in o_lists]), np.stack([i for _, i in o_lists]), K)

    ex = P.PeerExchange(aqr, NQ, K, S)
    try:
        assert (ex.world, ex.rank, ex.lo, ex.hi, ex.blk) == (1, 0, 0, NQ, NQ)
        searchers = [aqr.Searcher(ix, NQ, aqr.make_params(K, **m)) for ix in ixs]
        plain = [tuple(t.clone() for t in s_.run(qt)) for s_ in searchers]
        sd, si = aqr.merge_topk(torch.stack([d for _, d in plain]), torch.stack([i for i, _ in plain]))
        for step in range(3):  # both parities, the second one reused
            _, par = ex.begin()
            for s, sr in enumerate(searchers):
                assert sr.run(qt, out=ex.dest(0, s, par)) is None
            ld, li = ex.finish()
            md, mi = aqr.merge_topk(ld, li)
            torch.cuda.synchronize()
            ex.check()
            for s in range(S):  # the lists landed where the layout says, bit for bit
                assert torch.equal(li[s], plain[s][0]) and torch.equal(ld[s], plain[s][1])
            assert torch.equal(mi, si) and torch.equal(md, sd)
            np.testing.assert_array_equal(mi.cpu().numpy(), oi)
            np.testing.assert_allclose(md.cpu().numpy(), od, rtol=1e-5)
        del ld, li
    finally:
        ex.close()
        for ix in ixs:
            ix.free()


def _ipc_worker(rank, world, port, out_dir):
    import os
    import torch
    import torch.distributed as dist
    import paper_2602_21600_b200 as aqr
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ex = None
    try:
        # both processes share the one GPU: each maps the other's allocation through the CUDA IPC
        # handle (aqr_peer_open).  No kernel ever waits on the other process: the host barrier
        # orders the signal kernels before the waits, so every wait finds its flags set
        ex = P.PeerExchange(aqr, 8, 4, world, timeout_s=5.0)
        for step in range(2):
            _, par = ex.begin()
            # "search output": this rank's list of each owner's block, a recognisable pattern
            for o in range(world):
                lo, hi, _ = P.block_range(8, world, o)
                src_i = (torch.arange((hi - lo) * 4, dtype=torch.int32, device="cuda") + 1000 * rank + 100 * step)
                src_d = src_i.to(torch.float32) / 8
                p_i, p_d = ex.dest(o, rank, par)
                for ptr, src in ((p_i, src_i), (p_d, src_d)):
                    raw = aqr.PeerBuffer(ptr, src.numel() * 4, True)  # view only (never closed): a mapped address
                    raw.tensor(src.dtype, tuple(src.shape)).copy_(src)
            torch.cuda.synchronize()
            flags = [p.ptr + ex.lay["flags"] for p in ex.peers]
            aqr.peer_signal(flags, rank, ex.step)
            torch.cuda.synchronize()
            dist.barrier()
            aqr.peer_wait(flags[rank], world, ex.step, ex.timeout_ns, ex.status)
            torch.cuda.synchronize()
            ex.check()
            shape = (world, ex.blk, 4)
            li = ex.local.tensor(torch.int32, shape, ex.lay["ids"][par]).cpu().numpy()
            ld = ex.local.tensor(torch.float32, shape, ex.lay["dist"][par]).cpu().numpy()
            np.save(os.path.join(out_dir, f"s{step}_r{rank}_i.npy"), li)
            np.save(os.path.join(out_dir, f"s{step}_r{rank}_d.npy"), ld)
            dist.barrier()
    finally:
        if ex is not None:
            ex.close()
        dist.destroy_process_group()


def test_ipc_mapping_between_two_processes(tmp_path):
    """aqr_peer_open / aqr_peer_close and stores through the mapped pointers, two processes on the
    one GPU (handle exchange over gloo)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    mp.spawn(_ipc_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for step in range(2):
        for owner in range(world):
            li = np.load(tmp_path / f"s{step}_r{owner}_i.npy")
            ld = np.load(tmp_path / f"s{step}_r{owner}_d.npy")
            for src in range(world):  # list `src` of owner's block was written by process `src`
                want = np.arange(4 * 4, dtype=np.int32).reshape(4, 4) + 1000 * src + 100 * step
                np.testing.assert_array_equal(li[src], want)
                np.testing.assert_array_equal(ld[src], want.astype(np.float32) / 8)
