"""One TurboSpec decode step on device: lookup -> choose-k -> verify -> update.

Listing 1 for the PLD method: Propose (prompt lookup, fixed
length) -> GetVerificationLen = ArgMaxGoodput over the retrieved lengths ->
Score (the target forward: NOT here; its probability rows are synthetic inputs) ->
Accept (rejection sampling) -> UpdateGlobalAcceptance.  Every stage is one libtsv
launch on the caller's stream, with the real data dependencies kept: choose-k reads
the lookup's proposal lengths and the current alpha, and the alpha update reads the
verify's accepted counts; the next step's choose-k reads that alpha.  No host sync.

This module only wires buffers and launches (plumbing); all arithmetic is in the
sm_100a kernels.  Inputs rotate over ``sets`` to keep the timed region out of L2.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any, List, Optional

import torch

from . import tsv

# Defaults of the step's configuration (not arithmetic): the SPEC.md desk latency profiles
# (ctx_ms_per_tok, batched_ms_per_tok, fixed_ms) -- SPEC.md:50, 59-60 (target), 69 (draft) --
# and the Philox seed of the synthetic workloads.
DESK_TARGET = (0.001, 0.05, 2.0)
DESK_DRAFT = (0.0001, 0.005, 0.2)
DEFAULT_SEED = 240614066


@dataclass
class StepInputs:
    """The step's device inputs.  ``verify[s]`` is any object carrying the tsv_verify_args arrays
    of rotation set s as attributes: p, q (or None), row_offsets, draft_tokens, request_ids."""
    verify: List[Any]                      # one per rotation set (device)
    ctx: List[torch.Tensor]                # int32 contexts per set (device)
    ctx_offsets: List[torch.Tensor]        # int32 [B+1] per set (device)
    ctx_len: List[torch.Tensor]            # int32 [B] per set (device)
    k_max: int
    n_min: int = 1
    n_max: int = 4
    k_fixed: int = 5
    target: tuple = DESK_TARGET
    draft: tuple = DESK_DRAFT
    pld_cost_ms: float = 0.05
    kv_free_slots: int = -1
    seed: int = DEFAULT_SEED

    @property
    def B(self) -> int:
        """Largest batch over the rotation sets (buffer sizing; a strong-scaling rank's share of the
        batch can differ per set)."""
        return max(self.B_of(s) for s in range(self.sets))

    def B_of(self, s: int) -> int:
        return int(self.verify[s].row_offsets.numel()) - 1

    @property
    def sets(self) -> int:
        return len(self.verify)

    def input_bytes(self, s: int) -> int:
        """Bytes of one set's inputs (what an end-to-end call copies host -> device)."""
        vb = self.verify[s]
        n = vb.p.numel() * 4 + (0 if vb.q is None else vb.q.numel() * 4)
        n += (vb.row_offsets.numel() + vb.draft_tokens.numel() + vb.request_ids.numel()) * 4
        n += (self.ctx[s].numel() + self.ctx_offsets[s].numel() + self.ctx_len[s].numel()) * 4
        return n


class SpecStep:
    """Preallocated outputs + the step's launches; eager ``run`` or CUDA-graph ``capture``/``replay``.

    fused=False (default): tsv_propose_lookup, tsv_goodput_choose_k, tsv_verify_accept_update
    -- 5 kernels chained with PDL (the alpha update is an extra CTA of verify's emit kernel).
    fused=True: tsv_propose_lookup_choose_k (the lookup CTA that finishes last runs choose-k)
    + tsv_verify_accept_update, 4 kernels.  Identical outputs (tests/test_gpu_parity.py);
    the last-CTA handshake costs more than the kernel boundary it saves on B200.

    comm (request-sharded): this rank holds a disjoint part of one batch (global
    request ids) and alpha / k* are global -- one server over the ranks.
      tsv.P2PComm: tsv_goodput_choose_k_p2p (sums exchanged over NVLink peer memory inside the
        kernel) and tsv_verify_accept_update_p2p (the update CTA exchanges (sum m, sum t)):
        still 5 kernels per step, no NCCL launch;
      tsv.Comm (NCCL): partial -> ncclAllReduce -> finalize for both, 10 launches.
    k*, every k_i, every emitted token and alpha equal one device holding the whole batch."""

    def __init__(self, inp: StepInputs, device="cuda", alpha0: float = 0.7, chunk: int = 0, fused: bool = False,
                 comm=None, lookup_ready: bool = True, early_trigger: bool = True):
        self.inp = inp
        # the contexts are inputs of the step that no kernel of the step writes (prepared before the step,
        # like a serving engine's input buffers): TSV_LOOKUP_INPUTS_READY lets the lookup search them
        # while the previous step's last kernel drains (include/tsv.h states the contract)
        self.lookup_flags = tsv.LOOKUP_INPUTS_READY if lookup_ready else 0
        B, K = inp.B, inp.k_max
        dev = torch.device(device)
        self.alpha = torch.full((1,), alpha0, dtype=torch.float64, device=dev)
        self.proposals = torch.empty((B, inp.k_fixed), dtype=torch.int32, device=dev)
        self.proposal_len = torch.empty(B, dtype=torch.int32, device=dev)
        self.k_star = torch.empty(1, dtype=torch.int32, device=dev)
        self.goodput = torch.empty(inp.k_fixed + 1, dtype=torch.float64, device=dev)
        self.k_req = torch.empty(B, dtype=torch.int32, device=dev)
        self.num_accepted = torch.empty(B, dtype=torch.int32, device=dev)
        self.out_tokens = torch.empty((B, K + 1), dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.counter = tsv.lookup_choose_scratch(dev)  # fused lookup + choose-k
        # 1: alpha is final.  The verify + update call resets it and sets it once alpha is written; the
        # fused lookup + choose-k of the next step waits for it (it may start in the race's tail)
        self.alpha_ready = torch.ones(1, dtype=torch.int32, device=dev)
        self.fused = fused
        self.comm = comm
        self.p2p = comm is not None and not isinstance(comm, tsv.Comm)
        if fused and comm is not None:
            raise ValueError("the fused lookup + choose-k has no request-sharded variant")
        self.sums_ws = torch.zeros(tsv.gp_sums_len(inp.k_fixed), dtype=torch.int64, device=dev)
        self.upd_ws = torch.zeros(2, dtype=torch.int64, device=dev)
        self.args = []
        for vb in inp.verify:
            # the batch's row_offsets / drafts / request ids are inputs of the step, never written by
            # the step's own kernels (the proposer's output goes through the target forward first)
            # the next kernel after the verify call is the next step's lookup: with INPUTS_READY it
            # reads only the contexts (never written by a step kernel) before its wait, so the emit
            # may let it launch early (TSV_VERIFY_EARLY_TRIGGER): it searches in the race's tail
            # (the fused lookup + choose-k reads alpha, which this call's update CTA writes, before its
            # wait: it waits for the alpha_ready word the update sets, tsv_verify_accept_update_ex)
            early = lookup_ready and early_trigger
            flags = tsv.VERIFY_META_READY | (tsv.VERIFY_EARLY_TRIGGER if early else 0)
            a = tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids,
                                     inp.seed, 0, K, self.num_accepted, self.out_tokens, self.status,
                                     chunk=chunk, flags=flags)
            self.args.append(a)
        ws_bytes = max(tsv.tsv_verify_workspace_size(a) for a in self.args)
        self.workspace = tsv.alloc_workspace(ws_bytes, dev)
        for a in self.args:
            a.workspace = self.workspace.data_ptr()
            a.workspace_bytes = self.workspace.numel()
        self.graph: Optional[torch.cuda.CUDAGraph] = None

    @property
    def launches_per_step(self) -> int:
        if self.comm is not None and not self.p2p:
            return 10  # lookup, 3 x choose-k (partial, NCCL, finalize), 3 x verify, 3 x update
        return 4 if self.fused else 5

    def _choose_k(self, s, st):
        inp, L = self.inp, tsv.lib()
        args = (self.alpha.data_ptr(), 0, inp.ctx_len[s].data_ptr(), self.proposal_len.data_ptr(), inp.B_of(s),
                inp.k_fixed, tsv.POLICY_PLD, tsv.LatencyModel(*inp.target), tsv.LatencyModel(*inp.draft),
                float(inp.pld_cost_ms), int(inp.kv_free_slots), self.k_star.data_ptr(), self.goodput.data_ptr(),
                self.k_req.data_ptr())
        if self.comm is None:
            tsv._check(L.tsv_goodput_choose_k(*args, st))
        elif self.p2p:
            tsv._check(L.tsv_goodput_choose_k_p2p(*args, self.comm.handle, self.status.data_ptr(), st))
        else:
            tsv._check(L.tsv_goodput_choose_k_sharded(*args, self.sums_ws.data_ptr(), self.comm.handle, st))

    def _verify_update(self, a, s, st):
        L = tsv.lib()
        if self.comm is None:
            tsv._check(L.tsv_verify_accept_update(tsv.ctypes.byref(a), self.alpha.data_ptr(), 0, 0.9, tsv.EST_TESTED, st))
        elif self.p2p:
            tsv._check(L.tsv_verify_accept_update_p2p(tsv.ctypes.byref(a), self.alpha.data_ptr(), 0, 0.9,
                                                      tsv.EST_TESTED, self.comm.handle, st))
        else:
            tsv._check(L.tsv_verify_accept(tsv.ctypes.byref(a), st))
            tsv._check(L.tsv_update_acceptance_sharded(self.alpha.data_ptr(), self.num_accepted.data_ptr(),
                                                       self.inp.verify[s].row_offsets.data_ptr(), self.inp.B_of(s), 0.9,
                                                       tsv.EST_TESTED, self.upd_ws.data_ptr(), self.comm.handle, st))

    def run(self, step: int, stream=None):
        """Launch one decode step on ``stream`` (default: current)."""
        inp = self.inp
        s = step % inp.sets
        st = tsv._stream(stream)
        L = tsv.lib()
        if self.fused:
            tsv._check(L.tsv_propose_lookup_choose_k_ex(
                inp.ctx[s].data_ptr(), inp.ctx_offsets[s].data_ptr(), inp.B_of(s), inp.n_min, inp.n_max, inp.k_fixed,
                self.proposals.data_ptr(), self.proposal_len.data_ptr(), self.alpha.data_ptr(), 0,
                inp.ctx_len[s].data_ptr(), tsv.LatencyModel(*inp.target), float(inp.pld_cost_ms),
                int(inp.kv_free_slots), self.k_star.data_ptr(), self.goodput.data_ptr(), self.k_req.data_ptr(),
                self.counter.data_ptr(), self.status.data_ptr(),
                self.alpha_ready.data_ptr() if self.lookup_flags else None, self.lookup_flags, st))
            a = self.args[s]
            a.step = step & 0xFFFFFFFF
            tsv._check(L.tsv_verify_accept_update_ex(tsv.ctypes.byref(a), self.alpha.data_ptr(), 0, 0.9,
                                                     tsv.EST_TESTED, self.alpha_ready.data_ptr(), st))
            return
        tsv._check(L.tsv_propose_lookup_ex(inp.ctx[s].data_ptr(), inp.ctx_offsets[s].data_ptr(), inp.B_of(s),
                                           inp.n_min, inp.n_max, inp.k_fixed, self.proposals.data_ptr(),
                                           self.proposal_len.data_ptr(), self.status.data_ptr(), self.lookup_flags, st))
        self._choose_k(s, st)
        a = self.args[s]
        a.step = step & 0xFFFFFFFF
        self._verify_update(a, s, st)

    def run_component(self, name: str, step: int, stream=None):
        """One launch of a single step component (timing breakdown only)."""
        inp = self.inp
        s = step % inp.sets
        st = tsv._stream(stream)
        L = tsv.lib()
        if name == "lookup":  # flags 0: back-to-back READY lookups would overlap each other entirely
            tsv._check(L.tsv_propose_lookup_ex(inp.ctx[s].data_ptr(), inp.ctx_offsets[s].data_ptr(), inp.B_of(s),
                                               inp.n_min, inp.n_max, inp.k_fixed, self.proposals.data_ptr(),
                                               self.proposal_len.data_ptr(), self.status.data_ptr(), 0, st))
        elif name == "choose_k":
            self._choose_k(s, st)
        elif name == "verify":
            a = self.args[s]
            a.step = step & 0xFFFFFFFF
            tsv._check(L.tsv_verify_accept(tsv.ctypes.byref(a), st))
        elif name == "verify_update":
            a = self.args[s]
            a.step = step & 0xFFFFFFFF
            self._verify_update(a, s, st)
        elif name == "update":
            tsv._check(L.tsv_update_acceptance(self.alpha.data_ptr(), 0, self.num_accepted.data_ptr(),
                                               inp.verify[s].row_offsets.data_ptr(), inp.B_of(s), 0.9,
                                               tsv.EST_TESTED, st))
        else:
            raise ValueError(name)

    def capture(self, steps):
        """Capture ``steps`` consecutive decode steps into one CUDA graph."""
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up outside capture (lazy module loading)
            self.run(steps[0])
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.reset_state()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for t in steps:
                self.run(t)
        self.graph = g
        self.steps_in_graph = len(steps)

    def replay(self):
        self.graph.replay()

    def reset_state(self, alpha0: float = 0.7):
        self.alpha.fill_(alpha0)
        self.alpha_ready.fill_(1)
        self.status.zero_()

    def outputs(self):
        return {"proposals": self.proposals, "proposal_len": self.proposal_len, "k_star": self.k_star,
                "goodput": self.goodput, "k_req": self.k_req, "num_accepted": self.num_accepted,
                "out_tokens": self.out_tokens, "alpha": self.alpha, "status": self.status}
