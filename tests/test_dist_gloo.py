"""Multi-rank host logic on CPU with the gloo backend (world_size 2).

Covers what the N > 1 bench path does around the kernels: max-over-ranks timing,
sum-over-ranks token counts, broadcast of the 128-byte NCCL unique id, the all-gather of the 64-byte
CUDA IPC handles of the peer-memory buffers, and the
request / vocab partitions (global request ids => identical Philox streams)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_14066_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = pdist.max_over_ranks(1.5 + rank)
        s = pdist.sum_over_ranks(10 * (rank + 1))
        blob = bytes(range(128)) if rank == 0 else b"\x00" * 128
        got = pdist.broadcast_bytes(blob)
        k = np.random.Generator(np.random.PCG64(3)).integers(0, 9, 256)
        parts = pdist.partition_requests(k, world)
        handles = pdist.exchange_handles(bytes([rank]) * 64, rank, world)  # peer-memory handle exchange
        q.put((rank, t, s, got, parts, handles))
    finally:
        dist.destroy_process_group()


def test_two_rank_reductions_and_broadcast():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, s, got, parts, handles in res:
        assert handles == [bytes([r]) * 64 for r in range(world)]
        assert t == 2.5
        assert s == 30.0
        assert got == bytes(range(128))
        assert parts == res[0][4]


def test_partition_requests_balanced_and_contiguous():
    rng = np.random.Generator(np.random.PCG64(1))
    for world in (1, 2, 4, 8):
        for trial in range(20):
            k = rng.integers(0, 9, int(rng.integers(world, 600)))
            parts = pdist.partition_requests(k, world)
            assert parts[0][0] == 0 and parts[-1][1] == k.size
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            w = 2 * k + 1
            loads = [w[lo:hi].sum() for lo, hi in parts]
            assert max(loads) - min(loads) <= 2 * (2 * 8 + 1)


def test_vocab_shards_cover_and_align():
    for V in (32000, 128256, 13, 4099):
        for G in (1, 2, 4, 8):
            sh = pdist.vocab_shards(V, G)
            assert sh[0][0] == 0
            assert sum(n for _, n in sh) == V
            assert all(lo % 4 == 0 for lo, _ in sh)
            assert all(a[0] + a[1] == b[0] for a, b in zip(sh, sh[1:]))


def _slice_worker(rank, world, port, q):
    """Each rank takes its partition of one synthetic batch with request_slice / context_slice (the
    strong-scaling split of bench.py); the all-gathered slices must rebuild the whole batch."""
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        vb = synth.make_verify_batch(B=23, V=64, k_max=8, lam=0.7, seed=5)
        ctx, offs = synth.make_contexts(B=23, L=40, V=64, seed=5, ragged=True)
        lo, hi = pdist.partition_requests(vb.k.numpy(), world)[rank]
        p, qq, ro, d, rid = pdist.request_slice(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, lo, hi)
        c, o = pdist.context_slice(torch.tensor(ctx), torch.tensor(offs), lo, hi)
        mine = (lo, hi) + tuple(t.numpy().copy() for t in (p, qq, ro, d, rid, c, o))
        allp = [None] * world
        dist.all_gather_object(allp, mine)  # (numpy: tensors do not cross the spawn queue)
        q.put((rank, allp, tuple(t.numpy() for t in (vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids)),
               ctx, offs))
    finally:
        dist.destroy_process_group()


def test_two_rank_request_slices_rebuild_the_batch():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_slice_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, allp, (P, Q, RO, D, RID), c0, o0 = res[0]
    B = RO.size - 1
    assert allp[0][0] == 0 and allp[-1][1] == B and allp[0][1] == allp[1][0]
    cat = lambda i: np.concatenate([a[i] for a in allp])  # noqa: E731
    assert np.array_equal(cat(2), P) and np.array_equal(cat(3), Q)
    assert np.array_equal(cat(5), D) and np.array_equal(cat(6), RID)  # global request ids kept
    base = 0
    for a in allp:  # offsets rebased to 0 and consistent with the rows held
        assert a[4][0] == 0 and a[4][-1] == a[2].shape[0] and a[3].shape[0] == a[2].shape[0] - (a[1] - a[0])
        assert np.array_equal(a[4] + base, RO[a[0]:a[1] + 1])
        base += a[2].shape[0]
    assert np.array_equal(cat(7), c0)
    cb = 0
    for a in allp:
        assert np.array_equal(a[8] + cb, o0[a[0]:a[1] + 1])
        cb += a[7].size
