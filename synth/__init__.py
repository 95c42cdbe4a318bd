"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONLY thing the oracle side (tests) and the CUDA side
(bench, tests) share.  It holds none of the method's arithmetic: it draws
probability rows, drafts, ragged lengths and token contexts with torch's own
seeded generators; no acceptance test, race, lookup or goodput step is here.

Recipe:
  * p rows: RN32(softmax_f64(sigma * z)), z ~ N(0,1), sigma = 3  (p_max ~ 0.09, H ~ 6 nats)
  * q rows: RN32(lam * p + (1 - lam) * r), r an independent softmax row; the
    acceptance sum_v min(p, q) ~= lam  (paper's rates 0.53-0.92)
  * drafts x_j ~ q_j (or uniform-random when q is one-hot / absent)
  * k_i ~ U{0..k_max} (ragged verification lengths, config 2)
  * PLD contexts: Zipf(1.1) tokens over V plus copy spans (start w.p. 0.3 per
    position, length ~ Geometric(mean 16), copied from a uniform earlier offset),
    imitating the repetition PLD exploits
Seeds: seed = 240614066 by default; request ids 0..B-1 (global).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

DEFAULT_SEED = 240614066


@dataclass
class VerifyBatch:
    p: torch.Tensor            # float32 [R_p, ld]
    q: Optional[torch.Tensor]  # float32 [R_q, ld] or None (one-hot drafts)
    row_offsets: torch.Tensor  # int32 [B+1]
    draft_tokens: torch.Tensor  # int32 [R_q] (global ids)
    request_ids: torch.Tensor  # int32 (bit pattern of uint32) [B]
    k: torch.Tensor            # int32 [B]
    vocab: int
    k_max: int

    @property
    def B(self) -> int:
        return int(self.row_offsets.numel() - 1)

    @property
    def rows_p(self) -> int:
        return int(self.p.shape[0])

    def to(self, device) -> "VerifyBatch":
        mv = lambda t: None if t is None else t.to(device)
        return VerifyBatch(mv(self.p), mv(self.q), mv(self.row_offsets), mv(self.draft_tokens),
                           mv(self.request_ids), mv(self.k), self.vocab, self.k_max)


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    return g


def softmax_rows(n: int, V: int, sigma: float, g: torch.Generator, device, ld: int) -> torch.Tensor:
    """n rows of RN32(softmax_f64(sigma * z)), padded to ld columns with zeros."""
    out = torch.zeros((n, ld), dtype=torch.float32, device=device)
    step = max(1, (1 << 25) // max(V, 1))  # bound the float64 temporary
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        z = torch.randn((r1 - r0, V), generator=g, device=device, dtype=torch.float64)
        out[r0:r1, :V] = torch.softmax(sigma * z, dim=1).to(torch.float32)
    return out


def make_verify_batch(B: int, V: int, k_max: int, lam: float = 0.7, sigma: float = 3.0,
                      seed: int = DEFAULT_SEED, device="cpu", dense_q: bool = True,
                      k_fixed: Optional[int] = None, ld: Optional[int] = None,
                      k_list=None, request_id_base: int = 0) -> VerifyBatch:
    """Config-2/4-shaped verify inputs (ragged k_i ~ U{0..k_max} unless fixed)."""
    g = _gen(seed, device)
    ld = ld if ld is not None else (V + 3) // 4 * 4
    assert ld >= V and ld % 4 == 0
    if k_list is not None:
        k = torch.as_tensor(k_list, dtype=torch.int32).to(device)
    elif k_fixed is not None:
        k = torch.full((B,), int(k_fixed), dtype=torch.int32, device=device)
    else:
        k = torch.randint(0, k_max + 1, (B,), generator=g, device=device, dtype=torch.int32)
    row_offsets = torch.zeros(B + 1, dtype=torch.int32, device=device)
    row_offsets[1:] = torch.cumsum(k + 1, 0).to(torch.int32)
    R_p = int(row_offsets[-1].item()) if B > 0 else 0
    R_q = R_p - B
    p_all = softmax_rows(R_p, V, sigma, g, device, ld)
    # q rows are mixes of the p row at the same position and an independent row
    q = None
    # index of the p row matching each q row: request i, position j -> row_offsets[i] + j
    req_of_q = torch.repeat_interleave(torch.arange(B, device=device), k.to(torch.int64))
    pos_of_q = torch.arange(R_q, device=device) - (row_offsets[:-1].to(torch.int64) - torch.arange(B, device=device))[req_of_q]
    prow_of_q = row_offsets[:-1].to(torch.int64)[req_of_q] + pos_of_q
    if dense_q and R_q > 0:
        r = softmax_rows(R_q, V, sigma, g, device, ld)
        q = (lam * p_all[prow_of_q].to(torch.float64) + (1.0 - lam) * r.to(torch.float64)).to(torch.float32)
        del r
        drafts = torch.multinomial(q[:, :V], 1, generator=g).squeeze(1).to(torch.int32) if R_q else \
            torch.zeros(0, dtype=torch.int32, device=device)
    elif dense_q:
        q = torch.zeros((0, ld), dtype=torch.float32, device=device)
        drafts = torch.zeros(0, dtype=torch.int32, device=device)
    else:
        # one-hot drafts (PLD / top-1): take the target's likely token w.p. lam else uniform
        if R_q > 0:
            top = torch.multinomial(p_all[prow_of_q][:, :V], 1, generator=g).squeeze(1)
            unif = torch.randint(0, V, (R_q,), generator=g, device=device)
            coin = torch.rand(R_q, generator=g, device=device) < lam
            drafts = torch.where(coin, top, unif).to(torch.int32)
        else:
            drafts = torch.zeros(0, dtype=torch.int32, device=device)
    rids = (torch.arange(B, dtype=torch.int64, device=device) + request_id_base).to(torch.int32)
    return VerifyBatch(p_all, q, row_offsets, drafts, rids, k, V, k_max)


def make_logits_batch(B: int, V: int, k_max: int, lam: float = 0.7, sigma: float = 3.0,
                      seed: int = DEFAULT_SEED, device="cpu", dense_q: bool = True, ld: Optional[int] = None,
                      k_list=None) -> VerifyBatch:
    """The same batch as make_verify_batch with p and q given as LOGITS (NEXT 1): natural logs
    of the probability rows (a valid logit vector of each row; padding columns stay 0)."""
    vb = make_verify_batch(B, V, k_max, lam=lam, sigma=sigma, seed=seed, device=device, dense_q=dense_q, ld=ld,
                           k_list=k_list)
    vb.p[:, :V] = torch.log(vb.p[:, :V])
    if vb.q is not None:
        vb.q[:, :V] = torch.log(vb.q[:, :V])
    return vb


def make_contexts(B: int, L: int, V: int = 32000, seed: int = DEFAULT_SEED, ragged: bool = False,
                  zipf_a: float = 1.1, copy_prob: float = 0.3, copy_mean: float = 16.0):
    """PLD contexts: returns (ctx int32 [sum L_i], ctx_offsets int32 [B+1]) as numpy arrays."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lens = rng.integers(0, L + 1, B) if ragged else np.full(B, L)
    out = []
    for i in range(B):
        n = int(lens[i])
        toks = ((rng.zipf(zipf_a, n) - 1) % V).astype(np.int32)
        starts = rng.random(n) < copy_prob
        glen = rng.geometric(1.0 / copy_mean, n)
        pos = 1
        while pos < n:
            if starts[pos]:
                src = int(rng.integers(0, pos))
                ln = min(int(glen[pos]), n - pos)
                for t in range(ln):  # overlapping copies allowed (src + t may reach pos)
                    toks[pos + t] = toks[src + t]
                pos += ln
            else:
                pos += 1
        out.append(toks)
    offsets = np.zeros(B + 1, np.int32)
    offsets[1:] = np.cumsum([len(t) for t in out])
    ctx = np.concatenate(out) if out else np.zeros(0, np.int32)
    return ctx.astype(np.int32), offsets


def make_goodput_instance(B: int, k_max: int = 8, seed: int = DEFAULT_SEED, ctx_lo: int = 128,
                          ctx_hi: int = 4096, cap: Optional[int] = None):
    """Config-5 instance: ctx_len_i ~ U[ctx_lo, ctx_hi], cap_i = k_max (or given)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ctx_len = rng.integers(ctx_lo, ctx_hi + 1, B).astype(np.int32)
    caps = np.full(B, k_max if cap is None else cap, np.int32)
    return ctx_len, caps


def make_step_inputs(B: int, V: int, L: int, k_max: int = 8, seed: int = DEFAULT_SEED, device="cuda",
                     sets: int = 1, lam: float = 0.7):
    """A SpecStep's inputs (paper_2406_14066_b200.step.StepInputs) from this module's generators:
    `sets` rotation sets of a config-2-shaped verify batch and config-3-shaped PLD contexts."""
    from paper_2406_14066_b200.step import StepInputs  # lazy: only the container type
    vbs, ctxs, offs, lens = [], [], [], []
    for s in range(sets):
        vbs.append(make_verify_batch(B=B, V=V, k_max=k_max, lam=lam, seed=seed + 1000 * s, device=device))
        c, o = make_contexts(B=B, L=L, V=V, seed=seed + 1000 * s)
        ctxs.append(torch.tensor(c, device=device))
        offs.append(torch.tensor(o, device=device))
        lens.append(torch.tensor(np.diff(o).astype(np.int32), device=device))
    return StepInputs(vbs, ctxs, offs, lens, k_max, seed=seed)


# Latency profiles: (ctx_ms_per_tok, batched_ms_per_tok, fixed_ms)
SPEC_DESK_TARGET = (0.001, 0.05, 2.0)
SPEC_DESK_DRAFT = (0.0001, 0.005, 0.2)
H100_CASE_TARGET = (1.5625e-4, 0.024, 4.2)   # derived from PAPER.md:971 (7.4 ms at batch 50)
H100_CASE_DRAFT = (1.1e-5, 0.002, 1.25)
