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
