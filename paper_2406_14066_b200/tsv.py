"""Thin ctypes binding of libtsv.so (include/tsv.h) -- argument marshalling only.

Every function has the C entry point's name and forwards torch CUDA tensors as raw
device pointers plus the current CUDA stream.  No computation happens here: every
step of the path runs in the sm_100a kernels of libtsv.so.  If the library is not
built the import fails loudly (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSV_LIB_PATH") or os.path.join(_HERE, "lib", "libtsv.so")  # override: experiments only

TSV_OK = 0
STATUS_NAMES = {1: "TSV_ERR_INVALID_ARG", 2: "TSV_ERR_CUDA", 3: "TSV_ERR_NCCL",
                4: "TSV_ERR_UNSUPPORTED_DEVICE", 5: "TSV_ERR_WORKSPACE"}
DEVSTATUS_BAD_TOKEN = 1
DEVSTATUS_BAD_K = 2
DEVSTATUS_NO_WEIGHT = 4
DEVSTATUS_P2P_TIMEOUT = 8
DEVSTATUS_BAD_CONTEXT = 16
DEVSTATUS_WAIT_TIMEOUT = 32
VERIFY_NO_PRUNE = 1
VERIFY_SHARD_DENSE = 2
VERIFY_RACE_ONLY = 4  # measurement: the race kernel alone over a previous call's workspace
VERIFY_META_READY = 8  # row_offsets/drafts/request_ids not written by the preceding kernel on the stream
VERIFY_P2P_FUSED = 16  # peer-memory vocab sharding: race items push their chunk keys (no keys kernel)
VERIFY_EARLY_TRIGGER = 32  # the emit kernel lets the next kernel launch before the race completes (tsv.h)
LOOKUP_INPUTS_READY = 1  # tsv_propose_lookup_ex: ctx/ctx_offsets not written by any kernel in flight
LOOKUP_CHOOSE_SCRATCH = 512  # TSV_LOOKUP_CHOOSE_SCRATCH
POLICY_DRAFT = 0
POLICY_PLD = 1
EST_TESTED = 0
EST_PROPOSED = 1
MAX_K = 15

EXPORTED = [
    "tsv_last_error", "tsv_abi_version", "tsv_propose_lookup", "tsv_verify_workspace_size",
    "tsv_workspace_clear", "tsv_verify_accept", "tsv_verify_shard_partial",
    "tsv_verify_shard_combine", "tsv_goodput_choose_k", "tsv_update_acceptance",
    "tsv_comm_get_unique_id", "tsv_comm_init", "tsv_comm_destroy",
    "tsv_verify_sharded_workspace_size", "tsv_verify_accept_sharded", "tsv_allreduce_i64",
    "tsv_propose_lookup_choose_k", "tsv_verify_accept_update", "tsv_debug_race_E", "tsv_debug_philox",
    "tsv_goodput_partial", "tsv_goodput_finalize", "tsv_goodput_choose_k_sharded", "tsv_update_partial",
    "tsv_update_finalize", "tsv_update_acceptance_sharded", "tsv_verify_shard_flags", "tsv_verify_shard_race",
    "tsv_verify_shard_emit", "tsv_verify_greedy", "tsv_verify_logits_workspace_size",
    "tsv_verify_accept_logits", "tsv_softmax_rows", "tsv_fit_latency_model", "tsv_sim_target",
    "tsv_context_append", "tsv_goodput_choose_k_batched", "tsv_debug_race_row",
    "tsv_p2p_buffer_size", "tsv_p2p_alloc", "tsv_p2p_free", "tsv_p2p_open", "tsv_p2p_close", "tsv_p2p_init",
    "tsv_p2p_destroy", "tsv_verify_accept_sharded_p2p", "tsv_verify_shard_p2p_phase", "tsv_allreduce_i64_p2p",
    "tsv_goodput_choose_k_p2p", "tsv_update_acceptance_p2p", "tsv_verify_accept_update_p2p",
    "tsv_propose_lookup_ex", "tsv_propose_lookup_choose_k_ex", "tsv_verify_accept_update_ex",
]


def gp_sums_len(k_max: int) -> int:
    """TSV_GP_SUMS(k_max): int64 words of a request-sharded goodput partial."""
    return 2 * (k_max + 1) + 4


class TsvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class VerifyArgs(ctypes.Structure):
    """Mirror of tsv_verify_args (include/tsv.h)."""
    _fields_ = [
        ("p", ctypes.c_void_p), ("q", ctypes.c_void_p), ("row_offsets", ctypes.c_void_p),
        ("draft_tokens", ctypes.c_void_p), ("request_ids", ctypes.c_void_p),
        ("num_accepted", ctypes.c_void_p), ("out_tokens", ctypes.c_void_p),
        ("device_status", ctypes.c_void_p), ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_uint64), ("ld", ctypes.c_int64), ("seed", ctypes.c_uint64),
        ("step", ctypes.c_uint32), ("B", ctypes.c_int32), ("k_max", ctypes.c_int32),
        ("rows_p", ctypes.c_int32), ("vocab", ctypes.c_int32), ("vocab_offset", ctypes.c_int32),
        ("vocab_global", ctypes.c_int32), ("chunk", ctypes.c_int32), ("flags", ctypes.c_int32),
        ("step_counts", ctypes.c_void_p),
    ]


class LatencyModel(ctypes.Structure):
    """Mirror of tsv_latency_model: Eq. forward-time coefficients (alpha, gamma, delta) in ms."""
    _fields_ = [("ctx_ms_per_tok", ctypes.c_double), ("batched_ms_per_tok", ctypes.c_double),
                ("fixed_ms", ctypes.c_double)]


SHARD_TUPLE_BYTES = 24  # sizeof(tsv_shard_tuple)


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtsv.so not built at {LIB_PATH}: run `python -m paper_2406_14066_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u64, f64, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                 ctypes.c_double, ctypes.c_size_t)
    sig = {
        "tsv_last_error": ([], ctypes.c_char_p),
        "tsv_abi_version": ([], ctypes.c_int),
        "tsv_propose_lookup": ([P, P, i32, i32, i32, i32, P, P, P, P], ctypes.c_int),
        "tsv_propose_lookup_ex": ([P, P, i32, i32, i32, i32, P, P, P, i32, P], ctypes.c_int),
        "tsv_verify_workspace_size": ([ctypes.POINTER(VerifyArgs), ctypes.POINTER(sz)], ctypes.c_int),
        "tsv_workspace_clear": ([P, sz, P], ctypes.c_int),
        "tsv_verify_accept": ([ctypes.POINTER(VerifyArgs), P], ctypes.c_int),
        "tsv_verify_shard_partial": ([ctypes.POINTER(VerifyArgs), P, P], ctypes.c_int),
        "tsv_verify_shard_combine": ([ctypes.POINTER(VerifyArgs), P, i32, P], ctypes.c_int),
        "tsv_goodput_choose_k": ([P, i32, P, P, i32, i32, i32, LatencyModel, LatencyModel, f64, i64,
                                  P, P, P, P], ctypes.c_int),
        "tsv_update_acceptance": ([P, i32, P, P, i32, f64, i32, P], ctypes.c_int),
        "tsv_comm_get_unique_id": ([P], ctypes.c_int),
        "tsv_comm_init": ([ctypes.POINTER(P), P, i32, i32], ctypes.c_int),
        "tsv_comm_destroy": ([P], ctypes.c_int),
        "tsv_verify_sharded_workspace_size": ([ctypes.POINTER(VerifyArgs), i32, ctypes.POINTER(sz)],
                                              ctypes.c_int),
        "tsv_verify_accept_sharded": ([ctypes.POINTER(VerifyArgs), P, P], ctypes.c_int),
        "tsv_allreduce_i64": ([P, sz, P, P], ctypes.c_int),
        "tsv_propose_lookup_choose_k": ([P, P, i32, i32, i32, i32, P, P, P, i32, P, LatencyModel, f64, i64,
                                         P, P, P, P, P, P], ctypes.c_int),
        "tsv_propose_lookup_choose_k_ex": ([P, P, i32, i32, i32, i32, P, P, P, i32, P, LatencyModel, f64, i64,
                                            P, P, P, P, P, P, i32, P], ctypes.c_int),
        "tsv_verify_accept_update_ex": ([ctypes.POINTER(VerifyArgs), P, i32, f64, i32, P, P], ctypes.c_int),
        "tsv_verify_accept_update": ([ctypes.POINTER(VerifyArgs), P, i32, f64, i32, P], ctypes.c_int),
        "tsv_debug_race_E": ([ctypes.c_uint32, ctypes.c_uint32, P, P], ctypes.c_int),
        "tsv_debug_philox": ([P, P, ctypes.c_uint32, P, i32, P], ctypes.c_int),
        "tsv_goodput_partial": ([P, i32, P, P, i32, i32, P, P], ctypes.c_int),
        "tsv_goodput_finalize": ([P, i32, i32, LatencyModel, LatencyModel, f64, i64, P, i32, P, P, P, P],
                                 ctypes.c_int),
        "tsv_goodput_choose_k_sharded": ([P, i32, P, P, i32, i32, i32, LatencyModel, LatencyModel, f64, i64,
                                          P, P, P, P, P, P], ctypes.c_int),
        "tsv_update_partial": ([P, P, i32, i32, P, P], ctypes.c_int),
        "tsv_update_finalize": ([P, P, f64, P], ctypes.c_int),
        "tsv_update_acceptance_sharded": ([P, P, P, i32, f64, i32, P, P, P], ctypes.c_int),
        "tsv_verify_shard_flags": ([ctypes.POINTER(VerifyArgs), P, P], ctypes.c_int),
        "tsv_verify_shard_race": ([ctypes.POINTER(VerifyArgs), P, P, P], ctypes.c_int),
        "tsv_verify_shard_emit": ([ctypes.POINTER(VerifyArgs), P, P, P], ctypes.c_int),
        "tsv_verify_greedy": ([ctypes.POINTER(VerifyArgs), P], ctypes.c_int),
        "tsv_verify_logits_workspace_size": ([ctypes.POINTER(VerifyArgs), ctypes.POINTER(sz)], ctypes.c_int),
        "tsv_verify_accept_logits": ([ctypes.POINTER(VerifyArgs), ctypes.c_float, P], ctypes.c_int),
        "tsv_softmax_rows": ([P, i64, i32, i32, ctypes.c_float, P, P], ctypes.c_int),
        "tsv_fit_latency_model": ([P, P, P, i32, ctypes.POINTER(LatencyModel), P], ctypes.c_int),
        "tsv_sim_target": ([P, i32, P, i32, P, i32, i64, i32, P, P, P, P, P], ctypes.c_int),
        "tsv_context_append": ([P, i32, i32, P, P, i32, P, P, P], ctypes.c_int),
        "tsv_goodput_choose_k_batched": ([P, P, P, P, i32, i32, i32, LatencyModel, LatencyModel, f64, i64,
                                          P, P, P, P], ctypes.c_int),
        "tsv_debug_race_row": ([P, P, i32, i32, P, P], ctypes.c_int),
        "tsv_p2p_buffer_size": ([i32, ctypes.POINTER(sz)], ctypes.c_int),
        "tsv_p2p_alloc": ([i32, ctypes.POINTER(P), P], ctypes.c_int),
        "tsv_p2p_free": ([P], ctypes.c_int),
        "tsv_p2p_open": ([P, ctypes.POINTER(P)], ctypes.c_int),
        "tsv_p2p_close": ([P], ctypes.c_int),
        "tsv_p2p_init": ([ctypes.POINTER(P), i32, i32, i32, P], ctypes.c_int),
        "tsv_p2p_destroy": ([P], ctypes.c_int),
        "tsv_verify_accept_sharded_p2p": ([ctypes.POINTER(VerifyArgs), P, P], ctypes.c_int),
        "tsv_verify_shard_p2p_phase": ([ctypes.POINTER(VerifyArgs), P, i32, P], ctypes.c_int),
        "tsv_allreduce_i64_p2p": ([P, i32, P, P, P], ctypes.c_int),
        "tsv_goodput_choose_k_p2p": ([P, i32, P, P, i32, i32, i32, LatencyModel, LatencyModel, f64, i64,
                                      P, P, P, P, P, P], ctypes.c_int),
        "tsv_update_acceptance_p2p": ([P, i32, P, P, i32, f64, i32, P, P, P], ctypes.c_int),
        "tsv_verify_accept_update_p2p": ([ctypes.POINTER(VerifyArgs), P, i32, f64, i32, P, P], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


_lib = _load()


def lib() -> ctypes.CDLL:
    return _lib


def _check(status: int):
    if status != TSV_OK:
        msg = _lib.tsv_last_error()
        raise TsvError(status, msg.decode() if msg else "")


def _ptr(t: Optional[torch.Tensor], rows_ok: bool = False) -> Optional[int]:
    """Device-accessible pointer of a contiguous tensor (rows_ok: a 2-D row-strided view is fine):
    a CUDA tensor, or a pinned host tensor, which the kernels read over PCIe (UVA zero-copy)."""
    if t is None:
        return None
    if not t.is_cuda and not t.is_pinned():
        raise ValueError("libtsv takes CUDA tensors or pinned host tensors; got pageable host memory")
    ok = t.is_contiguous() or (rows_ok and t.dim() == 2 and t.stride(1) == 1)
    if not ok:
        raise ValueError("libtsv takes contiguous tensors")
    return t.data_ptr()


def _dev(t: torch.Tensor) -> torch.device:
    """Where to allocate outputs / workspaces for an input tensor (pinned host inputs -> current GPU)."""
    return t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())


def _stream(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _want(t, dtype, numel, name):
    if t.dtype != dtype:
        raise ValueError(f"{name}: expected {dtype}, got {t.dtype}")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name}: expected >= {numel} elements, got {t.numel()}")


def tsv_abi_version() -> int:
    return _lib.tsv_abi_version()


# ----------------------------------------------------------------------------- lookup
def tsv_propose_lookup(ctx: torch.Tensor, ctx_offsets: torch.Tensor, n_min: int, n_max: int,
                       k_fixed: int, proposals: Optional[torch.Tensor] = None,
                       proposal_len: Optional[torch.Tensor] = None, device_status=None, stream=None,
                       flags: int = 0):
    """Prompt-lookup proposal.  Returns (proposals[B, k], proposal_len[B]).
    flags: LOOKUP_INPUTS_READY (tsv_propose_lookup_ex; include/tsv.h states the contract)."""
    B = ctx_offsets.numel() - 1
    _want(ctx, torch.int32, None, "ctx")
    _want(ctx_offsets, torch.int32, None, "ctx_offsets")
    dev = _dev(ctx_offsets)
    if proposals is None:
        proposals = torch.empty((B, k_fixed), dtype=torch.int32, device=dev)
    if proposal_len is None:
        proposal_len = torch.empty(B, dtype=torch.int32, device=dev)
    ctx_p = _ptr(ctx) if ctx.numel() else _ptr(ctx_offsets)  # any valid pointer when empty
    _check(_lib.tsv_propose_lookup_ex(ctx_p, _ptr(ctx_offsets), B, n_min, n_max, k_fixed,
                                      _ptr(proposals), _ptr(proposal_len), _ptr(device_status), int(flags),
                                      _stream(stream)))
    return proposals, proposal_len


# ----------------------------------------------------------------------------- verify
def make_verify_args(p, q, row_offsets, draft_tokens, request_ids, seed, step, k_max,
                     num_accepted, out_tokens, device_status=None, workspace=None,
                     vocab=None, vocab_offset=0, vocab_global=None, chunk=0, flags=0,
                     step_counts=None) -> VerifyArgs:
    B = row_offsets.numel() - 1
    _want(p, torch.float32, None, "p")
    if q is not None:
        _want(q, torch.float32, None, "q")
    _want(row_offsets, torch.int32, B + 1, "row_offsets")
    _want(draft_tokens, torch.int32, None, "draft_tokens")
    if request_ids.dtype not in (torch.int32, torch.uint32):
        raise ValueError("request_ids must be int32/uint32")
    _want(num_accepted, torch.int32, B, "num_accepted")
    _want(out_tokens, torch.int32, B * (k_max + 1), "out_tokens")
    V = int(p.shape[1]) if vocab is None else int(vocab)
    a = VerifyArgs()
    a.p = _ptr(p, rows_ok=True)
    a.q = _ptr(q, rows_ok=True)
    a.row_offsets = _ptr(row_offsets)
    a.draft_tokens = _ptr(draft_tokens) if draft_tokens.numel() else None
    a.request_ids = _ptr(request_ids)
    a.num_accepted = _ptr(num_accepted)
    a.out_tokens = _ptr(out_tokens)
    a.device_status = _ptr(device_status)
    a.workspace = _ptr(workspace)
    a.workspace_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    a.ld = int(p.stride(0))
    if q is not None and q.shape[0] > 0 and int(q.stride(0)) != a.ld:
        raise ValueError("p and q must share the row stride ld")
    a.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    a.step = int(step) & 0xFFFFFFFF
    a.B = B
    a.k_max = int(k_max)
    a.rows_p = int(p.shape[0])
    a.vocab = V
    a.vocab_offset = int(vocab_offset)
    a.vocab_global = int(vocab_global) if vocab_global is not None else V
    a.chunk = int(chunk)
    a.flags = int(flags)
    if step_counts is not None:
        _want(step_counts, torch.int64, 2, "step_counts")
    a.step_counts = _ptr(step_counts)
    return a


def tsv_verify_workspace_size(args: VerifyArgs) -> int:
    n = ctypes.c_size_t(0)
    _check(_lib.tsv_verify_workspace_size(ctypes.byref(args), ctypes.byref(n)))
    return int(n.value)


def tsv_workspace_clear(workspace: torch.Tensor, stream=None):
    _check(_lib.tsv_workspace_clear(_ptr(workspace), workspace.numel() * workspace.element_size(),
                                    _stream(stream)))


def alloc_workspace(nbytes: int, device) -> torch.Tensor:
    """A zero-filled workspace (the contract: zero once after allocation)."""
    return torch.zeros(max(16, (nbytes + 15) // 16 * 16), dtype=torch.uint8, device=device)


def tsv_verify_accept(p, q, row_offsets, draft_tokens, request_ids, seed, step, k_max,
                      num_accepted=None, out_tokens=None, device_status=None, workspace=None,
                      chunk=0, flags=0, vocab=None, step_counts=None, stream=None):
    """Rejection-sampling verify/accept.  Returns (num_accepted, out_tokens)."""
    B = row_offsets.numel() - 1
    dev = _dev(row_offsets)
    if num_accepted is None:
        num_accepted = torch.empty(B, dtype=torch.int32, device=dev)
    if out_tokens is None:
        out_tokens = torch.empty((B, k_max + 1), dtype=torch.int32, device=dev)
    a = make_verify_args(p, q, row_offsets, draft_tokens, request_ids, seed, step, k_max,
                         num_accepted, out_tokens, device_status, workspace, vocab=vocab,
                         chunk=chunk, flags=flags, step_counts=step_counts)
    if workspace is None and B > 0:
        workspace = alloc_workspace(tsv_verify_workspace_size(a), dev)
        a.workspace = workspace.data_ptr()
        a.workspace_bytes = workspace.numel()
    _check(_lib.tsv_verify_accept(ctypes.byref(a), _stream(stream)))
    return num_accepted, out_tokens


def tsv_verify_greedy(p, row_offsets, draft_tokens, k_max, num_accepted=None, out_tokens=None,
                      device_status=None, workspace=None, vocab=None, chunk=0, step_counts=None, stream=None):
    """Greedy (temperature-0) verify (reading R24).  Returns (num_accepted, out_tokens)."""
    B = row_offsets.numel() - 1
    dev = _dev(p)
    if num_accepted is None:
        num_accepted = torch.empty(B, dtype=torch.int32, device=dev)
    if out_tokens is None:
        out_tokens = torch.empty((B, k_max + 1), dtype=torch.int32, device=dev)
    rids = torch.zeros(max(B, 1), dtype=torch.int32, device=dev)  # unused by the greedy rule
    a = make_verify_args(p, None, row_offsets, draft_tokens, rids[:B] if B else rids, 0, 0, k_max,
                         num_accepted, out_tokens, device_status, workspace, vocab=vocab, chunk=chunk,
                         step_counts=step_counts)
    if workspace is None and B > 0:
        workspace = alloc_workspace(tsv_verify_workspace_size(a), dev)
        a.workspace = workspace.data_ptr()
        a.workspace_bytes = workspace.numel()
    _check(_lib.tsv_verify_greedy(ctypes.byref(a), _stream(stream)))
    return num_accepted, out_tokens


def tsv_verify_logits_workspace_size(args: VerifyArgs) -> int:
    n = ctypes.c_size_t(0)
    _check(_lib.tsv_verify_logits_workspace_size(ctypes.byref(args), ctypes.byref(n)))
    return int(n.value)


def tsv_verify_accept_logits(zp, zq, row_offsets, draft_tokens, request_ids, seed, step, k_max,
                             temperature=1.0, num_accepted=None, out_tokens=None, device_status=None,
                             workspace=None, vocab=None, chunk=0, flags=0, step_counts=None, stream=None):
    """Fused softmax-from-logits verify (reading R23).  Returns (num_accepted, out_tokens)."""
    B = row_offsets.numel() - 1
    dev = _dev(zp)
    if num_accepted is None:
        num_accepted = torch.empty(B, dtype=torch.int32, device=dev)
    if out_tokens is None:
        out_tokens = torch.empty((B, k_max + 1), dtype=torch.int32, device=dev)
    a = make_verify_args(zp, zq, row_offsets, draft_tokens, request_ids, seed, step, k_max,
                         num_accepted, out_tokens, device_status, workspace, vocab=vocab, chunk=chunk, flags=flags,
                         step_counts=step_counts)
    if workspace is None and B > 0:
        workspace = alloc_workspace(tsv_verify_logits_workspace_size(a), dev)
        a.workspace = workspace.data_ptr()
        a.workspace_bytes = workspace.numel()
    _check(_lib.tsv_verify_accept_logits(ctypes.byref(a), float(temperature), _stream(stream)))
    return num_accepted, out_tokens


def tsv_softmax_rows(z, temperature=1.0, vocab=None, out=None, stream=None):
    """Probabilities from logits rows (reading R23), fp32 [rows, ld]."""
    _want(z, torch.float32, None, "z")
    rows, ld = z.shape
    V = ld if vocab is None else int(vocab)
    if out is None:
        out = torch.empty_like(z)
    _check(_lib.tsv_softmax_rows(_ptr(z, rows_ok=True), int(z.stride(0)), V, rows, float(temperature), _ptr(out),
                                 _stream(stream)))
    return out


def tsv_verify_shard_partial(args: VerifyArgs, tuples_out: torch.Tensor, stream=None):
    _check(_lib.tsv_verify_shard_partial(ctypes.byref(args), _ptr(tuples_out), _stream(stream)))
    return tuples_out


def tsv_verify_shard_combine(args: VerifyArgs, gathered: torch.Tensor, num_shards: int, stream=None):
    _check(_lib.tsv_verify_shard_combine(ctypes.byref(args), _ptr(gathered), int(num_shards),
                                         _stream(stream)))


def tsv_verify_shard_flags(args: VerifyArgs, masks_out: torch.Tensor, stream=None):
    """Lazy sharding round 1: int64 [B] (owner bits << 32 | accept bits) of this shard's drafts."""
    _check(_lib.tsv_verify_shard_flags(ctypes.byref(args), _ptr(masks_out), _stream(stream)))


def tsv_verify_shard_race(args: VerifyArgs, masks: torch.Tensor, keys_out: torch.Tensor, stream=None):
    """Lazy sharding round 2: race row m_i (from the summed masks) -> int64 [2B] (key, fallback key)."""
    _check(_lib.tsv_verify_shard_race(ctypes.byref(args), _ptr(masks), _ptr(keys_out), _stream(stream)))


def tsv_verify_shard_emit(args: VerifyArgs, masks: torch.Tensor, keys: torch.Tensor, stream=None):
    """Emit from the summed masks and the max-reduced keys."""
    _check(_lib.tsv_verify_shard_emit(ctypes.byref(args), _ptr(masks), _ptr(keys), _stream(stream)))


def lookup_choose_scratch(device) -> torch.Tensor:
    """Zero-filled scratch for tsv_propose_lookup_choose_k."""
    return torch.zeros(LOOKUP_CHOOSE_SCRATCH // 8, dtype=torch.int64, device=device)


def tsv_propose_lookup_choose_k(ctx, ctx_offsets, n_min, n_max, k_fixed, alpha, ctx_len, target,
                                pld_cost_ms, counter, kv_free_slots=-1, alpha_per_request=None,
                                proposals=None, proposal_len=None, k_out=None, goodput_out=None,
                                k_per_request=None, device_status=None, stream=None, flags: int = 0,
                                alpha_ready=None):
    """Fused prompt lookup + PLD goodput selection.  ``counter``: device scratch of
    LOOKUP_CHOOSE_SCRATCH bytes (e.g. lookup_choose_scratch()), zeroed once.
    flags: LOOKUP_INPUTS_READY (tsv_propose_lookup_choose_k_ex; include/tsv.h states the contract).
    Returns (proposals, proposal_len, k_out, goodput_out)."""
    B = ctx_offsets.numel() - 1
    dev = _dev(ctx_offsets)
    if counter.numel() * counter.element_size() < LOOKUP_CHOOSE_SCRATCH:
        raise ValueError(f"counter scratch must hold {LOOKUP_CHOOSE_SCRATCH} bytes")
    if proposals is None:
        proposals = torch.empty((B, k_fixed), dtype=torch.int32, device=dev)
    if proposal_len is None:
        proposal_len = torch.empty(B, dtype=torch.int32, device=dev)
    if k_out is None:
        k_out = torch.empty(1, dtype=torch.int32, device=dev)
    if goodput_out is None:
        goodput_out = torch.empty(k_fixed + 1, dtype=torch.float64, device=dev)
    per = (alpha.numel() == B and B > 1) if alpha_per_request is None else bool(alpha_per_request)
    ctx_p = _ptr(ctx) if ctx.numel() else _ptr(ctx_offsets)
    _check(_lib.tsv_propose_lookup_choose_k_ex(ctx_p, _ptr(ctx_offsets), B, n_min, n_max, k_fixed,
                                               _ptr(proposals), _ptr(proposal_len), _ptr(alpha),
                                               1 if per else 0, _ptr(ctx_len), LatencyModel(*target),
                                               float(pld_cost_ms), int(kv_free_slots), _ptr(k_out),
                                               _ptr(goodput_out), _ptr(k_per_request), _ptr(counter),
                                               _ptr(device_status), _ptr(alpha_ready), int(flags), _stream(stream)))
    return proposals, proposal_len, k_out, goodput_out


def tsv_verify_accept_update(args: VerifyArgs, alpha, decay=0.9, estimator=EST_TESTED, per_request=False,
                             stream=None):
    """Fused verify/accept + acceptance update (alpha fp64 device, in place)."""
    _want(alpha, torch.float64, 1, "alpha")
    _check(_lib.tsv_verify_accept_update(ctypes.byref(args), _ptr(alpha), 1 if per_request else 0,
                                         float(decay), int(estimator), _stream(stream)))


# ----------------------------------------------------------------------------- goodput
def tsv_goodput_choose_k(alpha, ctx_len, cap, k_max, policy, target, draft=(0.0, 0.0, 0.0),
                         pld_cost_ms=0.0, kv_free_slots=-1, alpha_per_request=None, k_out=None,
                         goodput_out=None, k_per_request=None, stream=None):
    """ArgMaxGoodput (Listing 2).  Returns (k_out[1], goodput[k_max+1], k_per_request)."""
    B = ctx_len.numel()
    dev = _dev(ctx_len)
    _want(alpha, torch.float64, 1, "alpha")
    _want(ctx_len, torch.int32, None, "ctx_len")
    _want(cap, torch.int32, B, "cap")
    per = (alpha.numel() == B and B > 1) if alpha_per_request is None else bool(alpha_per_request)
    if k_out is None:
        k_out = torch.empty(1, dtype=torch.int32, device=dev)
    if goodput_out is None:
        goodput_out = torch.empty(k_max + 1, dtype=torch.float64, device=dev)
    _check(_lib.tsv_goodput_choose_k(_ptr(alpha), 1 if per else 0, _ptr(ctx_len), _ptr(cap), B,
                                     int(k_max), int(policy), LatencyModel(*target),
                                     LatencyModel(*draft), float(pld_cost_ms), int(kv_free_slots),
                                     _ptr(k_out), _ptr(goodput_out), _ptr(k_per_request),
                                     _stream(stream)))
    return k_out, goodput_out, k_per_request


def tsv_goodput_choose_k_batched(alpha, ctx_len, cap, inst_offsets, k_max, policy, target, draft=(0.0, 0.0, 0.0),
                                 pld_cost_ms=0.0, kv_free_slots=-1, k_out=None, goodput_out=None,
                                 k_per_request=None, stream=None):
    """n_inst independent ArgMaxGoodput problems in one launch.  Returns (k_out[n], goodput[n, k_max+1])."""
    n = inst_offsets.numel() - 1
    dev = _dev(ctx_len)
    _want(alpha, torch.float64, n, "alpha")
    if k_out is None:
        k_out = torch.empty(n, dtype=torch.int32, device=dev)
    if goodput_out is None:
        goodput_out = torch.empty((n, k_max + 1), dtype=torch.float64, device=dev)
    _check(_lib.tsv_goodput_choose_k_batched(_ptr(alpha), _ptr(ctx_len), _ptr(cap), _ptr(inst_offsets), n,
                                             int(k_max), int(policy), LatencyModel(*target), LatencyModel(*draft),
                                             float(pld_cost_ms), int(kv_free_slots), _ptr(k_out),
                                             _ptr(goodput_out), _ptr(k_per_request), _stream(stream)))
    return k_out, goodput_out


def tsv_update_acceptance(alpha, num_accepted, row_offsets, decay=0.9, estimator=EST_TESTED,
                          per_request=False, stream=None):
    """UpdateGlobalAcceptance, in place on ``alpha`` (fp64 device)."""
    B = num_accepted.numel()
    _want(alpha, torch.float64, B if per_request else 1, "alpha")
    _want(num_accepted, torch.int32, None, "num_accepted")
    _want(row_offsets, torch.int32, B + 1, "row_offsets")
    _check(_lib.tsv_update_acceptance(_ptr(alpha), 1 if per_request else 0, _ptr(num_accepted),
                                      _ptr(row_offsets), B, float(decay), int(estimator),
                                      _stream(stream)))
    return alpha


# ------------------------------------------------------------- request-sharded goodput / update
def tsv_goodput_partial(alpha, ctx_len, cap, k_max, alpha_per_request=None, sums=None, stream=None):
    """This rank's exact int64 batch sums for ArgMaxGoodput (TSV_GP_SUMS(k_max) words)."""
    B = ctx_len.numel()
    dev = _dev(ctx_len)
    _want(ctx_len, torch.int32, None, "ctx_len")
    _want(cap, torch.int32, B, "cap")
    per = (alpha.numel() == B and B > 1) if alpha_per_request is None else bool(alpha_per_request)
    if sums is None:
        sums = torch.empty(gp_sums_len(k_max), dtype=torch.int64, device=dev)
    _check(_lib.tsv_goodput_partial(_ptr(alpha), 1 if per else 0, _ptr(ctx_len), _ptr(cap), B, int(k_max),
                                    _ptr(sums), _stream(stream)))
    return sums


def tsv_goodput_finalize(sums, k_max, policy, target, draft=(0.0, 0.0, 0.0), pld_cost_ms=0.0,
                         kv_free_slots=-1, cap=None, k_out=None, goodput_out=None, k_per_request=None,
                         stream=None):
    """ArgMaxGoodput on (rank-summed) sums; k_per_request = min(k*, cap) for the local requests."""
    dev = _dev(sums)
    _want(sums, torch.int64, gp_sums_len(k_max), "sums")
    if k_out is None:
        k_out = torch.empty(1, dtype=torch.int32, device=dev)
    if goodput_out is None:
        goodput_out = torch.empty(k_max + 1, dtype=torch.float64, device=dev)
    B_local = 0 if cap is None else cap.numel()
    _check(_lib.tsv_goodput_finalize(_ptr(sums), int(k_max), int(policy), LatencyModel(*target),
                                     LatencyModel(*draft), float(pld_cost_ms), int(kv_free_slots), _ptr(cap),
                                     B_local, _ptr(k_out), _ptr(goodput_out), _ptr(k_per_request),
                                     _stream(stream)))
    return k_out, goodput_out, k_per_request


def tsv_update_partial(num_accepted, row_offsets, estimator=EST_TESTED, sums=None, stream=None):
    """This rank's (sum m_i, sum t_i) as int64[2]."""
    B = num_accepted.numel()
    _want(row_offsets, torch.int32, B + 1, "row_offsets")
    if sums is None:
        sums = torch.empty(2, dtype=torch.int64, device=_dev(num_accepted))
    _check(_lib.tsv_update_partial(_ptr(num_accepted), _ptr(row_offsets), B, int(estimator), _ptr(sums),
                                   _stream(stream)))
    return sums


def tsv_update_finalize(alpha, sums, decay=0.9, stream=None):
    _want(alpha, torch.float64, 1, "alpha")
    _want(sums, torch.int64, 2, "sums")
    _check(_lib.tsv_update_finalize(_ptr(alpha), _ptr(sums), float(decay), _stream(stream)))
    return alpha


def tsv_fit_latency_model(ctx_tokens, batched_tokens, ms):
    """Host-side OLS latency fit (reading R25).  Returns ((ctx, batched, fixed) ms coefficients, R^2)."""
    c = np.ascontiguousarray(ctx_tokens, np.float64)
    b = np.ascontiguousarray(batched_tokens, np.float64)
    t = np.ascontiguousarray(ms, np.float64)
    out = LatencyModel()
    r2 = ctypes.c_double(0.0)
    _check(_lib.tsv_fit_latency_model(c.ctypes.data, b.ctypes.data, t.ctypes.data, int(t.size), ctypes.byref(out),
                                      ctypes.byref(r2)))
    return (out.ctx_ms_per_tok, out.batched_ms_per_tok, out.fixed_ms), float(r2.value)


# ----------------------------------------------------------------------------- comm
class Comm:
    """NCCL communicator owned by libtsv; the unique id travels over torch.distributed."""

    def __init__(self, rank: int, world: int, group=None):
        import torch.distributed as dist
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _check(_lib.tsv_comm_get_unique_id(ctypes.cast(uid, ctypes.c_void_p)))
        obj = [bytes(uid)]
        if dist.is_initialized() and world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        raw = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        _check(_lib.tsv_comm_init(ctypes.byref(h), ctypes.cast(raw, ctypes.c_void_p), int(rank), int(world)))
        self.handle = h
        self.rank, self.world = rank, world

    def close(self):
        if self.handle:
            _check(_lib.tsv_comm_destroy(self.handle))
            self.handle = None


class P2PComm:
    """Peer-memory exchange for the lazy vocab-sharded verify (tsv_verify_accept_sharded_p2p).

    Every rank allocates its symmetric buffer in libtsv (cudaMalloc, zero-filled) and
    exports its 64-byte CUDA IPC handle; the handles travel over torch.distributed
    (all_gather_object) and each rank maps its peers' buffers (cudaIpcOpenMemHandle).
    Host-side plumbing only: the exchange itself runs in the kernels."""

    def __init__(self, rank: int, world: int, B_max: int, group=None):
        import torch.distributed as dist
        self.rank, self.world, self.B_max = int(rank), int(world), int(B_max)
        own = ctypes.c_void_p()
        hnd = (ctypes.c_uint8 * 64)()
        _check(_lib.tsv_p2p_alloc(self.B_max, ctypes.byref(own), ctypes.cast(hnd, ctypes.c_void_p)))
        self.own = own
        from . import dist as pdist
        handles = pdist.exchange_handles(bytes(hnd), self.rank, self.world, group)
        self.opened = []
        self.handle = None
        bufs = (ctypes.c_void_p * self.world)()
        err = None
        try:
            for g, h in enumerate(handles):
                if g == self.rank:
                    bufs[g] = own.value
                    continue
                raw = (ctypes.c_uint8 * 64).from_buffer_copy(h)
                ptr = ctypes.c_void_p()
                _check(_lib.tsv_p2p_open(ctypes.cast(raw, ctypes.c_void_p), ctypes.byref(ptr)))
                self.opened.append(ptr)
                bufs[g] = ptr.value
            h = ctypes.c_void_p()
            _check(_lib.tsv_p2p_init(ctypes.byref(h), self.rank, self.world, self.B_max,
                                     ctypes.cast(bufs, ctypes.c_void_p)))
            self.handle = h
        except TsvError as e:  # e.g. no peer access between these GPUs
            err = e
        # every rank learns whether every rank mapped its peers (this all-reduce also orders every
        # mapping before anyone's first store), so all ranks fail -- or proceed -- together
        if self.world > 1 and dist.is_initialized():
            dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else None
            ok = pdist.min_over_ranks(0.0 if err else 1.0, device=dev, group=group)
        else:
            ok = 0.0 if err else 1.0
        if ok < 1.0:
            self.close()
            raise TsvError(2, f"P2PComm: peer mapping failed on some rank ({err or 'another rank'})")

    def close(self):
        if self.handle:
            _check(_lib.tsv_p2p_destroy(self.handle))
            self.handle = None
        for p in self.opened:
            _check(_lib.tsv_p2p_close(p))
        self.opened = []
        if self.own:
            _check(_lib.tsv_p2p_free(self.own))
            self.own = None


class P2PLoopback:
    """G virtual ranks on one device (tests): one local buffer per rank, every rank's peer table
    holds all of them.  Drive with tsv_verify_shard_p2p_phase: all ranks phase 0, then 1, then 2."""

    def __init__(self, world: int, B_max: int):
        self.world, self.B_max = int(world), int(B_max)
        self.bufs = []
        for _ in range(self.world):
            b = ctypes.c_void_p()
            _check(_lib.tsv_p2p_alloc(self.B_max, ctypes.byref(b), None))
            self.bufs.append(b)
        table = (ctypes.c_void_p * self.world)(*[b.value for b in self.bufs])
        self.handles = []
        for g in range(self.world):
            h = ctypes.c_void_p()
            _check(_lib.tsv_p2p_init(ctypes.byref(h), g, self.world, self.B_max, ctypes.cast(table, ctypes.c_void_p)))
            self.handles.append(h)

    def close(self):
        for h in self.handles:
            _check(_lib.tsv_p2p_destroy(h))
        for b in self.bufs:
            _check(_lib.tsv_p2p_free(b))
        self.handles, self.bufs = [], []


class P2PLoopbackRank:
    """Rank g of a P2PLoopback, usable wherever a P2PComm is (tests)."""

    def __init__(self, lb: "P2PLoopback", g: int):
        self.handle, self.rank, self.world = lb.handles[g], g, lb.world


def tsv_verify_accept_update_p2p(args: VerifyArgs, alpha, p2p, decay=0.9, estimator=EST_TESTED, per_request=False,
                                 stream=None):
    """Verify/accept + the request-sharded global alpha update, the (sum m, sum t) exchange done by
    the update CTA beside the race over peer memory (tsv_verify_accept_update_p2p)."""
    _check(_lib.tsv_verify_accept_update_p2p(ctypes.byref(args), _ptr(alpha), 1 if per_request else 0, float(decay),
                                             int(estimator), p2p.handle, _stream(stream)))


def tsv_verify_accept_sharded_p2p(args: VerifyArgs, p2p, stream=None):
    h = p2p.handle if hasattr(p2p, "handle") else p2p
    _check(_lib.tsv_verify_accept_sharded_p2p(ctypes.byref(args), h, _stream(stream)))


def tsv_verify_shard_p2p_phase(args: VerifyArgs, handle, phase: int, stream=None):
    _check(_lib.tsv_verify_shard_p2p_phase(ctypes.byref(args), handle, int(phase), _stream(stream)))


def tsv_verify_sharded_workspace_size(args: VerifyArgs, world: int) -> int:
    n = ctypes.c_size_t(0)
    _check(_lib.tsv_verify_sharded_workspace_size(ctypes.byref(args), int(world), ctypes.byref(n)))
    return int(n.value)


def tsv_verify_accept_sharded(args: VerifyArgs, comm: Comm, stream=None):
    _check(_lib.tsv_verify_accept_sharded(ctypes.byref(args), comm.handle, _stream(stream)))


def tsv_allreduce_i64_p2p(data: torch.Tensor, p2p, device_status=None, stream=None):
    """In-place exact int64 sum over the ranks through peer memory (tsv_allreduce_i64_p2p)."""
    _want(data, torch.int64, None, "data")
    _check(_lib.tsv_allreduce_i64_p2p(_ptr(data), int(data.numel()), p2p.handle, _ptr(device_status),
                                      _stream(stream)))


def tsv_goodput_choose_k_sharded(alpha, ctx_len, cap, k_max, policy, target, comm,
                                 draft=(0.0, 0.0, 0.0), pld_cost_ms=0.0, kv_free_slots=-1,
                                 alpha_per_request=None, k_out=None, goodput_out=None, k_per_request=None,
                                 sums_ws=None, device_status=None, stream=None):
    """Request-sharded ArgMaxGoodput: partial -> all-reduce(sum, int64) -> finalize.  comm: a Comm
    (ncclAllReduce inside tsv_goodput_choose_k_sharded) or a P2PComm (the single fused kernel
    tsv_goodput_choose_k_p2p)."""
    B = ctx_len.numel()
    dev = _dev(ctx_len)
    per = (alpha.numel() == B and B > 1) if alpha_per_request is None else bool(alpha_per_request)
    if k_out is None:
        k_out = torch.empty(1, dtype=torch.int32, device=dev)
    if goodput_out is None:
        goodput_out = torch.empty(k_max + 1, dtype=torch.float64, device=dev)
    if sums_ws is None:
        sums_ws = torch.empty(gp_sums_len(k_max), dtype=torch.int64, device=dev)
    if isinstance(comm, (P2PComm, P2PLoopbackRank)):  # one kernel: partial -> peer-memory sum -> finalize
        _check(_lib.tsv_goodput_choose_k_p2p(_ptr(alpha), 1 if per else 0, _ptr(ctx_len), _ptr(cap), B, int(k_max),
                                             int(policy), LatencyModel(*target), LatencyModel(*draft),
                                             float(pld_cost_ms), int(kv_free_slots), _ptr(k_out), _ptr(goodput_out),
                                             _ptr(k_per_request), comm.handle, _ptr(device_status), _stream(stream)))
        return k_out, goodput_out, k_per_request
    _check(_lib.tsv_goodput_choose_k_sharded(_ptr(alpha), 1 if per else 0, _ptr(ctx_len), _ptr(cap), B,
                                             int(k_max), int(policy), LatencyModel(*target),
                                             LatencyModel(*draft), float(pld_cost_ms), int(kv_free_slots),
                                             _ptr(k_out), _ptr(goodput_out), _ptr(k_per_request),
                                             _ptr(sums_ws), comm.handle, _stream(stream)))
    return k_out, goodput_out, k_per_request


def tsv_update_acceptance_sharded(alpha, num_accepted, row_offsets, comm, decay=0.9,
                                  estimator=EST_TESTED, sums_ws=None, device_status=None, stream=None):
    """Request-sharded global alpha update: partial -> all-reduce(sum, int64) -> finalize (NCCL Comm),
    or with a P2PComm the single kernel tsv_update_acceptance_p2p."""
    B = num_accepted.numel()
    if isinstance(comm, (P2PComm, P2PLoopbackRank)):
        _check(_lib.tsv_update_acceptance_p2p(_ptr(alpha), 0, _ptr(num_accepted), _ptr(row_offsets), B, float(decay),
                                              int(estimator), comm.handle, _ptr(device_status), _stream(stream)))
        return alpha
    if sums_ws is None:
        sums_ws = torch.empty(2, dtype=torch.int64, device=_dev(num_accepted))
    _check(_lib.tsv_update_acceptance_sharded(_ptr(alpha), _ptr(num_accepted), _ptr(row_offsets), B,
                                              float(decay), int(estimator), _ptr(sums_ws), comm.handle,
                                              _stream(stream)))
    return alpha


def tsv_allreduce_i64(data: torch.Tensor, comm: Comm, stream=None):
    _want(data, torch.int64, None, "data")
    _check(_lib.tsv_allreduce_i64(_ptr(data), data.numel(), comm.handle, _stream(stream)))
    return data


# ----------------------------------------------------------------------------- diagnostics
def tsv_debug_race_E(m_begin: int, n: int, out=None, device="cuda"):
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=device)
    _check(_lib.tsv_debug_race_E(int(m_begin), int(n), _ptr(out), _stream(None)))
    return out


def tsv_debug_race_row(w: torch.Tensor, words: torch.Tensor, prune: bool = True) -> int:
    """Packed race key of one row with injected Philox words (diagnostics)."""
    out = torch.zeros(1, dtype=torch.int64, device=w.device)
    _check(_lib.tsv_debug_race_row(_ptr(w), _ptr(words), int(w.numel()), 1 if prune else 0, _ptr(out),
                                   _stream(None)))
    return int(out.item()) & 0xFFFFFFFFFFFFFFFF


def tsv_debug_philox(ctr: torch.Tensor, key: torch.Tensor, race_variant: bool = False):
    n = ctr.numel() // 4
    out = torch.empty(4 * n, dtype=torch.int32, device=ctr.device)
    _check(_lib.tsv_debug_philox(_ptr(ctr), _ptr(key), n, _ptr(out), 1 if race_variant else 0, _stream(None)))
    return out
