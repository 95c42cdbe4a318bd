"""Pins for the closed-loop harness oracles (reading R26): the synthetic target rows and the
context-window append; and the world property the loop relies on -- the sampling verify keeps
each draft with probability alpha_true."""
import numpy as np
import pytest

import oracle
import synth

from loop_ref import run_oracle_loop


def test_sim_target_rows():
    props = np.array([[3, 1, 4, -1], [5, 9, 2, 6], [7, -1, -1, -1]], np.int32)
    kreq = np.array([3, 0, 1], np.int32)
    p, ro, d = oracle.sim_target(props, kreq, 0.75, 10)
    assert ro.tolist() == [0, 4, 5, 7] and d.tolist() == [3, 1, 4, 7]
    rest = np.float32((1 - 0.75) / 9)
    for r, x in [(0, 3), (1, 1), (2, 4), (5, 7)]:
        assert p[r, x] == np.float32(0.75) and (np.delete(p[r], x) == rest).all()
    for r in (3, 4, 6):  # bonus rows
        assert (p[r] == np.float32(0.1)).all()
    assert np.abs(p.astype(np.float64).sum(axis=1) - 1).max() < 1e-6


def test_acceptance_rate_is_alpha_true():
    # one draft per request, many requests and seeds: the fraction accepted estimates alpha_true
    B, V = 400, 64
    rng = np.random.Generator(np.random.PCG64(81))
    for a in (0.3, 0.9):
        props = rng.integers(0, V, (B, 1)).astype(np.int32)
        p, ro, d = oracle.sim_target(props, np.ones(B, np.int32), a, V)
        acc = 0
        for seed in range(10):
            na, _, _ = oracle.verify(p, None, ro, d, np.arange(B, dtype=np.uint32), seed, 0, 1)
            acc += int(na.sum())
        n = 10 * B
        assert abs(acc / n - a) < 4 * np.sqrt(a * (1 - a) / n)


def test_context_append_window():
    L = 6
    ctx = np.arange(12, dtype=np.int32)  # request 0: 0..5, request 1: 6..11
    out = np.array([[20, 21, 22], [30, -1, -1]], np.int32)
    na = np.array([2, 0], np.int32)
    new, cl = oracle.context_append(ctx, L, out, na, [100, 50])
    assert new.tolist() == [3, 4, 5, 20, 21, 22, 7, 8, 9, 10, 11, 30] and cl.tolist() == [103, 51]
    new, cl = oracle.context_append(ctx, L, out, np.array([-1, 0], np.int32), [100, 50])
    assert new[:6].tolist() == list(range(6)) and cl.tolist() == [100, 51]  # flagged request unchanged


def test_oracle_loop_tracks_alpha_true():
    B, L, V, K = 16, 128, 256, 5
    ctx, _ = synth.make_contexts(B=B, L=L, V=V, seed=3)
    steps = 40
    log, _, _ = run_oracle_loop(ctx, L, np.full(B, L, np.int32), 0.7, [0.9] * steps, steps, V, K,
                                synth.SPEC_DESK_TARGET, 0.05, seed=11)
    assert abs(log[-1]["alpha"] - 0.9) < 0.08
    for e in log:  # conservation: 1 <= m + 1 <= k_i + 1 tokens per request
        assert ((e["num_accepted"] >= 0) & (e["num_accepted"] <= e["k_req"])).all()
