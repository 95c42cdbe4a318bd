"""Host-side plumbing of the multi-GPU modes.

Request-sharded (independent units, no data-path collective): each rank owns a
contiguous range of requests with GLOBAL request ids, so Philox streams and hence
outputs are identical to a 1-GPU run (R6).  For a fixed global batch (strong
scaling) the ranges are balanced by the rows each request streams in the dense
worst case, 2k_i + 1.  Vocab-sharded: rank g owns a 4-aligned column range.
Timing: per-rank device time, reduced with MAX; token counts reduced with SUM.
Works with any torch.distributed backend (nccl on the GPU box, gloo in CPU tests).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def partition_requests(k: np.ndarray, world: int) -> List[Tuple[int, int]]:
    """Contiguous [lo, hi) request ranges, one per rank, balancing sum(2 k_i + 1)."""
    k = np.asarray(k, np.int64)
    n = k.size
    if world <= 1:
        return [(0, n)]
    w = 2 * k + 1
    c = np.concatenate([[0], np.cumsum(w)])
    total = c[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        j = int(np.searchsorted(c, target, side="left"))
        j = min(max(j, bounds[-1]), n)
        # pick the closer of j-1, j
        if j > bounds[-1] and abs(c[j - 1] - target) <= abs(c[j] - target):
            j -= 1
        bounds.append(max(j, bounds[-1]))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def vocab_shards(vocab: int, world: int) -> List[Tuple[int, int]]:
    """[offset, size) column shards with 4-aligned offsets (tsv_verify_args.vocab_offset % 4 == 0)."""
    quads = (vocab + 3) // 4
    out = []
    for g in range(world):
        q0 = quads * g // world
        q1 = quads * (g + 1) // world
        lo = 4 * q0
        hi = min(vocab, 4 * q1)
        out.append((lo, max(0, hi - lo)))
    return out


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def min_over_ranks(value: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t)
    return float(t.item())


def broadcast_bytes(blob: bytes, src: int = 0) -> bytes:
    """Broadcast an opaque blob (e.g. the 128-byte NCCL unique id) from ``src``."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return blob
    obj = [blob]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def exchange_handles(local: bytes, rank: int, world: int, group=None) -> list:
    """Every rank's blob (e.g. the 64-byte CUDA IPC handle of its peer-memory buffer) in rank
    order, via all_gather_object (any backend).  One rank: [local]."""
    import torch.distributed as dist
    if world <= 1 or not (dist.is_available() and dist.is_initialized()):
        return [local]
    out = [None] * world
    dist.all_gather_object(out, local, group=group)
    assert all(isinstance(b, bytes) and len(b) == len(local) for b in out), "handle exchange failed"
    assert out[rank] == local
    return out


def request_slice(p, q, row_offsets, draft_tokens, request_ids, lo: int, hi: int):
    """Requests [lo, hi) of one ragged verify batch as their own batch (views of the same storage):
    p rows row_offsets[lo] .. row_offsets[hi]-1, q rows / drafts shifted by the request index
    (packing row_offsets[i] - i), offsets rebased to 0.  Request ids stay GLOBAL (R6), so a rank's
    outputs equal the unsharded run's for its requests."""
    import torch
    ro = row_offsets.to(torch.int64)
    r0, r1 = int(ro[lo]), int(ro[hi])
    q0, q1 = r0 - lo, r1 - hi
    sub_ro = (row_offsets[lo:hi + 1] - row_offsets[lo]).contiguous()
    return (p[r0:r1], None if q is None else q[q0:q1], sub_ro, draft_tokens[q0:q1], request_ids[lo:hi])


def context_slice(ctx, ctx_offsets, lo: int, hi: int):
    """Contexts of requests [lo, hi) with offsets rebased to 0 (host or device tensors)."""
    c0, c1 = int(ctx_offsets[lo]), int(ctx_offsets[hi])
    return ctx[c0:c1], (ctx_offsets[lo:hi + 1] - ctx_offsets[lo])
