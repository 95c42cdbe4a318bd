"""Closed decode loop on the device (reading R26 in DESIGN.md).

One step = tsv_propose_lookup -> tsv_goodput_choose_k (PLD policy, cap = proposal lengths) ->
tsv_sim_target (synthetic target rows: each draft kept with probability alpha_true[t]) ->
tsv_verify_accept_update (one-hot drafts, alpha EWMA) -> tsv_context_append; every step also
logs k*, alpha and the accepted counts into device arrays.  All launches are asynchronous on one
stream, so ``capture`` records T steps as one CUDA graph that replays the controller's feedback
loop without a host round trip.  Marshalling only: every step runs in libtsv.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from . import tsv


class ClosedLoop:
    def __init__(self, ctx0: np.ndarray, L: int, ctx_len0: np.ndarray, V: int, K: int,
                 target: Sequence[float], pld_cost_ms: float, alpha_true: Sequence[float], alpha0: float = 0.7,
                 seed: int = 1, decay: float = 0.9, n_min: int = 1, n_max: int = 4, device="cuda"):
        dev = torch.device(device)
        self.B = B = int(np.asarray(ctx_len0).size)
        self.L, self.V, self.K, self.T = int(L), int(V), int(K), len(alpha_true)
        self.ld = (V + 3) // 4 * 4
        self.target = tsv.LatencyModel(*target)
        self.pld_cost_ms, self.seed, self.decay = float(pld_cost_ms), int(seed), float(decay)
        self.n_min, self.n_max = int(n_min), int(n_max)
        i32 = torch.int32
        self.ctx = [torch.tensor(np.asarray(ctx0, np.int32), device=dev), torch.empty(B * L, dtype=i32, device=dev)]
        self._init = (self.ctx[0].clone(), torch.tensor(np.asarray(ctx_len0, np.int32), device=dev), float(alpha0))
        self.ctx_offsets = torch.arange(0, (B + 1) * L, L, dtype=i32, device=dev)
        self.ctx_len = torch.tensor(np.asarray(ctx_len0, np.int32), device=dev)
        self.alpha = torch.full((1,), float(alpha0), dtype=torch.float64, device=dev)
        self.alpha_true = torch.tensor(np.asarray(alpha_true, np.float32), device=dev)
        self.proposals = torch.empty((B, K), dtype=i32, device=dev)
        self.proposal_len = torch.empty(B, dtype=i32, device=dev)
        self.k_star = torch.empty(1, dtype=i32, device=dev)
        self.goodput = torch.empty(K + 1, dtype=torch.float64, device=dev)
        self.k_req = torch.empty(B, dtype=i32, device=dev)
        self.rows_cap = B * (K + 1)
        self.p = torch.zeros((self.rows_cap, self.ld), dtype=torch.float32, device=dev)
        self.row_offsets = torch.zeros(B + 1, dtype=i32, device=dev)
        self.drafts = torch.zeros(max(1, B * K), dtype=i32, device=dev)
        self.row_info = torch.zeros(self.rows_cap, dtype=i32, device=dev)
        self.rids = torch.arange(B, dtype=i32, device=dev)
        self.num_accepted = torch.empty(B, dtype=i32, device=dev)
        self.out_tokens = torch.empty((B, K + 1), dtype=i32, device=dev)
        self.status = torch.zeros(1, dtype=i32, device=dev)
        # per-step logs
        self.log_k = torch.zeros(self.T, dtype=i32, device=dev)
        self.log_alpha = torch.zeros(self.T, dtype=torch.float64, device=dev)
        self.log_m = torch.zeros((self.T, B), dtype=i32, device=dev)
        self.log_kreq = torch.zeros((self.T, B), dtype=i32, device=dev)
        self.log_out = torch.zeros((self.T, B, K + 1), dtype=i32, device=dev)
        self.log_ctxlen = torch.zeros((self.T, B), dtype=i32, device=dev)
        self.log_plen = torch.zeros((self.T, B), dtype=i32, device=dev)
        self.args = []
        for t in range(self.T):
            a = tsv.make_verify_args(self.p, None, self.row_offsets, self.drafts, self.rids, self.seed, t, K,
                                     self.num_accepted, self.out_tokens, self.status, None, vocab=V)
            a.rows_p = self.rows_cap
            self.args.append(a)
        self.workspace = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(self.args[0]), dev)
        for a in self.args:
            a.workspace, a.workspace_bytes = self.workspace.data_ptr(), self.workspace.numel()
        self.graph: Optional[torch.cuda.CUDAGraph] = None

    def reset(self, stream=None):
        """Back to the initial contexts, context lengths and alpha (device copies; graph-capturable)."""
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
            self.ctx[0].copy_(self._init[0])
            self.ctx_len.copy_(self._init[1])
            self.alpha.fill_(self._init[2])

    def step(self, t: int, stream=None, log: bool = True):
        """Launch decode step t (reads window t % 2, writes the other)."""
        L_ = tsv.lib()
        st = tsv._stream(stream)
        B, K = self.B, self.K
        cin, cout = self.ctx[t % 2], self.ctx[(t + 1) % 2]
        tsv._check(L_.tsv_propose_lookup(cin.data_ptr(), self.ctx_offsets.data_ptr(), B, self.n_min, self.n_max, K,
                                         self.proposals.data_ptr(), self.proposal_len.data_ptr(),
                                         self.status.data_ptr(), st))
        tsv._check(L_.tsv_goodput_choose_k(self.alpha.data_ptr(), 0, self.ctx_len.data_ptr(),
                                           self.proposal_len.data_ptr(), B, K, tsv.POLICY_PLD, self.target,
                                           tsv.LatencyModel(0.0, 0.0, 0.0), self.pld_cost_ms, -1,
                                           self.k_star.data_ptr(), self.goodput.data_ptr(), self.k_req.data_ptr(), st))
        tsv._check(L_.tsv_sim_target(self.proposals.data_ptr(), K, self.k_req.data_ptr(), B,
                                     self.alpha_true[t:].data_ptr(), self.V, self.ld, self.rows_cap, self.p.data_ptr(),
                                     self.row_offsets.data_ptr(), self.drafts.data_ptr(), self.row_info.data_ptr(), st))
        tsv._check(L_.tsv_verify_accept_update(tsv.ctypes.byref(self.args[t]), self.alpha.data_ptr(), 0, self.decay,
                                               tsv.EST_TESTED, st))
        tsv._check(L_.tsv_context_append(cin.data_ptr(), self.L, B, self.out_tokens.data_ptr(),
                                         self.num_accepted.data_ptr(), K, cout.data_ptr(), self.ctx_len.data_ptr(), st))
        if not log:
            return
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
            self.log_k[t:t + 1].copy_(self.k_star)
            self.log_alpha[t:t + 1].copy_(self.alpha)
            self.log_m[t].copy_(self.num_accepted)
            self.log_kreq[t].copy_(self.k_req)
            self.log_out[t].copy_(self.out_tokens)
            self.log_ctxlen[t].copy_(self.ctx_len)
            self.log_plen[t].copy_(self.proposal_len)

    def run(self):
        """All T steps eagerly on the current stream."""
        for t in range(self.T):
            self.step(t)

    def capture(self, log: bool = True, with_reset: bool = False):
        """All T steps as one CUDA graph (replay() runs the whole closed loop).  with_reset: the graph
        starts from the initial state, so every replay repeats the same T steps (timing)."""
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                if with_reset:
                    self.reset(stream=side)
                for t in range(self.T):
                    self.step(t, stream=side, log=log)
        self.graph = g

    def logs(self):
        torch.cuda.synchronize()
        return {"k_star": self.log_k.cpu().numpy(), "alpha": self.log_alpha.cpu().numpy(),
                "num_accepted": self.log_m.cpu().numpy(), "k_req": self.log_kreq.cpu().numpy(),
                "out_tokens": self.log_out.cpu().numpy(), "ctx_len": self.log_ctxlen.cpu().numpy(),
                "proposal_len": self.log_plen.cpu().numpy()}
