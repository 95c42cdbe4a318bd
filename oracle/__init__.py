"""CPU oracle for the TurboSpec propose/verify/accept step -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct C (oracle.c) written from the paper
(arXiv 2406.14066, /root/reference/PAPER.md) and the readings in DESIGN.md §3.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It
shares no code with, and never imports, ``paper_2406_14066_b200``.

Functions (each cites its passage in oracle.c):
  philox4x32_10, u_acc, u_race, E, E_table  -- RNG and race uniforms (R6, R9)
  verify       -- rejection-sampling accept + residual/bonus race
  verify_greedy -- temperature-0 verify: keep drafts equal to the target argmax
  softmax_rows, verify_logits -- probabilities from logits (reading R23), then verify
  lookup       -- prompt-lookup n-gram proposal
  expected_len, forward_time, choose_k -- goodput adaptor
  update       -- moving-average acceptance update
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

STATUS_BAD_TOKEN = 1
STATUS_BAD_K = 2
STATUS_NO_WEIGHT = 4
POLICY_DRAFT = 0
POLICY_PLD = 1
EST_TESTED = 0
EST_PROPOSED = 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        cmd = ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, u32, u64, f64 = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                    ctypes.c_uint64, ctypes.c_double)
        lib.oracle_philox4x32_10.argtypes = [P, P, P]
        lib.oracle_philox4x32_10.restype = None
        lib.oracle_u_acc.argtypes = [u32]
        lib.oracle_u_acc.restype = ctypes.c_float
        lib.oracle_u_race.argtypes = [u32]
        lib.oracle_u_race.restype = ctypes.c_float
        lib.oracle_E.argtypes = [ctypes.c_float]
        lib.oracle_E.restype = ctypes.c_float
        lib.oracle_E_table.argtypes = [P]
        lib.oracle_E_table.restype = None
        lib.oracle_verify.argtypes = [P, P, i64, i32, P, P, P, u64, u32, i32, i32, P, P, P, P]
        lib.oracle_verify.restype = i32
        lib.oracle_verify_greedy.argtypes = [P, i64, i32, P, P, i32, i32, P, P]
        lib.oracle_verify_greedy.restype = i32
        lib.oracle_softmax_rows.argtypes = [P, i64, i32, i32, ctypes.c_float, P]
        lib.oracle_softmax_rows.restype = None
        lib.oracle_fit_latency.argtypes = [P, P, P, i32, P, P]
        lib.oracle_fit_latency.restype = i32
        lib.oracle_sim_target.argtypes = [P, i32, P, i32, ctypes.c_float, i32, i64, P, P, P]
        lib.oracle_sim_target.restype = None
        lib.oracle_context_append.argtypes = [P, i32, i32, P, P, i32, P, P]
        lib.oracle_context_append.restype = None
        lib.oracle_lookup.argtypes = [P, P, i32, i32, i32, i32, P, P]
        lib.oracle_lookup.restype = None
        lib.oracle_expected_len.argtypes = [f64, i32]
        lib.oracle_expected_len.restype = f64
        lib.oracle_forward_time.argtypes = [P, f64, f64]
        lib.oracle_forward_time.restype = f64
        lib.oracle_choose_k.argtypes = [P, i32, P, P, i32, i32, i32, P, P, f64, i64, P]
        lib.oracle_choose_k.restype = i32
        lib.oracle_update.argtypes = [P, i32, P, P, i32, f64, i32]
        lib.oracle_update.restype = None
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def philox4x32_10(ctr, key):
    lib = _load()
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib.oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def u_acc(x: int) -> float:
    return float(np.float32(_load().oracle_u_acc(int(x))))


def u_race(x: int) -> float:
    return float(np.float32(_load().oracle_u_race(int(x))))


def E(u: float) -> float:
    return float(np.float32(_load().oracle_E(float(u))))


def E_table() -> np.ndarray:
    """E(u) for every race uniform u = (2m+1) 2^-24, m = 0 .. 2^23-1."""
    out = np.zeros(1 << 23, np.float32)
    _load().oracle_E_table(_ptr(out))
    return out


def verify(p, q, row_offsets, draft_tokens, request_ids, seed, step, k_max,
           inj_u_acc=None, inj_E=None, vocab=None):
    """Returns (num_accepted[B], out_tokens[B, k_max+1], status).

    p: float32 [R_p, ld] (columns 0..V-1 used, V = p.shape[1] unless ``vocab`` differs);
    q: float32 [R_q, ld] or None (one-hot drafts)."""
    lib = _load()
    p = _c(p, np.float32)
    q = _c(q, np.float32)
    ro = _c(row_offsets, np.int32)
    dt = _c(draft_tokens, np.int32)
    if dt.size == 0:
        dt = np.zeros(1, np.int32)
    rid = _c(request_ids, np.uint32)
    B = ro.size - 1
    ld = p.shape[1]
    V = ld if vocab is None else int(vocab)
    assert 0 < V <= ld
    if q is not None:
        assert q.shape[1] == ld
    ia = _c(inj_u_acc, np.float32)
    ie = _c(inj_E, np.float32)
    na = np.zeros(B, np.int32)
    out = np.zeros((B, k_max + 1), np.int32)
    st = lib.oracle_verify(_ptr(p), _ptr(q), ld, V, _ptr(ro), _ptr(dt), _ptr(rid),
                           int(seed), int(step), B, int(k_max), _ptr(ia), _ptr(ie),
                           _ptr(na), _ptr(out))
    return na, out, int(st)


def verify_greedy(p, row_offsets, draft_tokens, k_max, vocab=None):
    """Greedy (temperature-0) verify: returns (num_accepted[B], out_tokens[B, k_max+1], status)."""
    lib = _load()
    p = _c(p, np.float32)
    ro = _c(row_offsets, np.int32)
    dt = _c(draft_tokens, np.int32)
    if dt.size == 0:
        dt = np.zeros(1, np.int32)
    B = ro.size - 1
    ld = p.shape[1]
    V = ld if vocab is None else int(vocab)
    na = np.zeros(B, np.int32)
    out = np.zeros((B, k_max + 1), np.int32)
    st = lib.oracle_verify_greedy(_ptr(p), ld, V, _ptr(ro), _ptr(dt), B, int(k_max), _ptr(na), _ptr(out))
    return na, out, int(st)


def softmax_rows(z, temperature=1.0, vocab=None):
    """Reading R23: fp32 exp, fp64 row sum, p = RN32(e * RN32(1/S)).  z: float32 [rows, ld]."""
    lib = _load()
    z = _c(z, np.float32)
    rows, ld = z.shape
    V = ld if vocab is None else int(vocab)
    out = np.zeros_like(z)
    lib.oracle_softmax_rows(_ptr(z), ld, V, rows, float(temperature), _ptr(out))
    return out


def verify_logits(zp, zq, row_offsets, draft_tokens, request_ids, seed, step, k_max, temperature=1.0,
                  vocab=None):
    """Fused-logits verify (NEXT 1): softmax_rows of the target and draft logits, then verify."""
    p = softmax_rows(zp, temperature, vocab)
    q = None if zq is None else softmax_rows(zq, temperature, vocab)
    return verify(p, q, row_offsets, draft_tokens, request_ids, seed, step, k_max, vocab=vocab)


def fit_latency(ctx_tokens, batched_tokens, ms):
    """Reading R25: OLS of ms on (ctx, batched, 1) with clamp-and-refit of negative coefficients.
    Returns ((ctx_ms_per_tok, batched_ms_per_tok, fixed_ms), r2); raises ValueError on error."""
    lib = _load()
    c = _c(ctx_tokens, np.float64)
    b = _c(batched_tokens, np.float64)
    t = _c(ms, np.float64)
    out = np.zeros(3, np.float64)
    r2 = np.zeros(1, np.float64)
    st = lib.oracle_fit_latency(_ptr(c), _ptr(b), _ptr(t), int(t.size), _ptr(out), _ptr(r2))
    if st == 1:
        raise ValueError("TooFewSamples")
    if st == 2:
        raise ValueError("DegenerateDesign")
    return tuple(float(x) for x in out), float(r2[0])


def sim_target(proposals, k_req, alpha_true, V, ld=None):
    """Closed-loop synthetic target (reading R26): returns (p [R, ld], row_offsets [B+1], drafts [R-B])."""
    lib = _load()
    pr = _c(proposals, np.int32)
    B, K = pr.shape
    kr = _c(k_req, np.int32)
    ld = V if ld is None else ld
    R = int((kr + 1).sum())
    p = np.zeros((max(R, 1), ld), np.float32)
    ro = np.zeros(B + 1, np.int32)
    d = np.zeros(max(R - B, 1), np.int32)
    lib.oracle_sim_target(_ptr(pr), K, _ptr(kr), B, float(alpha_true), int(V), ld, _ptr(p), _ptr(ro), _ptr(d))
    return p[:R], ro, d[:R - B]


def context_append(ctx, L, out_tokens, num_accepted, ctx_len):
    """Window append (reading R26): returns (new ctx [B*L], new ctx_len [B])."""
    lib = _load()
    c = _c(ctx, np.int32)
    ot = _c(out_tokens, np.int32)
    na = _c(num_accepted, np.int32)
    B = na.size
    out = np.zeros_like(c)
    cl = np.array(ctx_len, np.int32).copy()
    lib.oracle_context_append(_ptr(c), int(L), B, _ptr(ot), _ptr(na), int(ot.shape[1] - 1), _ptr(out), _ptr(cl))
    return out, cl


def lookup(ctx, ctx_offsets, n_min, n_max, K):
    lib = _load()
    c = _c(ctx, np.int32)
    if c.size == 0:
        c = np.zeros(1, np.int32)
    off = _c(ctx_offsets, np.int32)
    B = off.size - 1
    props = np.zeros((B, K), np.int32)
    plen = np.zeros(B, np.int32)
    lib.oracle_lookup(_ptr(c), _ptr(off), B, int(n_min), int(n_max), int(K), _ptr(props), _ptr(plen))
    return props, plen


def expected_len(alpha: float, k: int) -> float:
    return _load().oracle_expected_len(float(alpha), int(k))


def forward_time(model, n_context, n_batched) -> float:
    m = _c(model, np.float64)
    return _load().oracle_forward_time(_ptr(m), float(n_context), float(n_batched))


def choose_k(alpha, ctx_len, cap, k_max, policy, target, draft, pld_cost_ms=0.0,
             kv_free_slots=-1):
    """Returns (k*, goodput[k_max+1]).  ``alpha`` scalar => global, array => per request."""
    lib = _load()
    a = np.atleast_1d(np.asarray(alpha, np.float64))
    per_req = 1 if np.ndim(alpha) > 0 else 0
    cl = _c(ctx_len, np.int32)
    cp = _c(cap, np.int32)
    B = cl.size
    if per_req:
        assert a.size == B
    t = _c(target, np.float64)
    d = _c(draft if draft is not None else (0.0, 0.0, 0.0), np.float64)
    g = np.zeros(k_max + 1, np.float64)
    k = lib.oracle_choose_k(_ptr(a), per_req, _ptr(cl), _ptr(cp), B, int(k_max), int(policy),
                            _ptr(t), _ptr(d), float(pld_cost_ms), int(kv_free_slots), _ptr(g))
    return int(k), g


def update(alpha, num_accepted, row_offsets, decay=0.9, estimator=EST_TESTED):
    """Returns the updated alpha (scalar in => scalar out; array in => per-request)."""
    lib = _load()
    per_req = 1 if np.ndim(alpha) > 0 else 0
    a = np.array(np.atleast_1d(alpha), np.float64)
    na = _c(num_accepted, np.int32)
    ro = _c(row_offsets, np.int32)
    lib.oracle_update(_ptr(a), per_req, _ptr(na), _ptr(ro), na.size, float(decay), int(estimator))
    return a if per_req else float(a[0])
