"""Closed decode loop on the GPU (NEXT 4): bit-exact against the CPU reference loop composed of
oracle functions, and the controller's adaptation properties."""
import sys
import os

import numpy as np
import pytest
import torch

import oracle
import synth

sys.path.insert(0, os.path.dirname(__file__))
from loop_ref import run_oracle_loop  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def loop_mod():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2406_14066_b200 import loop
    return loop


def _make(loop_mod, B, L, V, K, alpha_true, seed=5, target=synth.SPEC_DESK_TARGET, alpha0=0.7, ctx_len0=None):
    ctx, _ = synth.make_contexts(B=B, L=L, V=V, seed=seed)
    cl = np.full(B, L, np.int32) if ctx_len0 is None else np.asarray(ctx_len0, np.int32)
    lp = loop_mod.ClosedLoop(ctx, L, cl, V, K, target, 0.05, alpha_true, alpha0=alpha0, seed=seed)
    return lp, ctx, cl


@pytest.mark.parametrize("graph", [False, True])
def test_closed_loop_bit_exact_vs_oracle(loop_mod, graph):
    B, L, V, K, T = 12, 128, 256, 5, 30
    at = [0.9] * 15 + [0.4] * 15
    lp, ctx, cl = _make(loop_mod, B, L, V, K, at)
    if graph:
        lp.capture()
        lp.graph.replay()
    else:
        lp.run()
    g = lp.logs()
    ref, rctx, rcl = run_oracle_loop(ctx, L, cl, 0.7, at, T, V, K, synth.SPEC_DESK_TARGET, 0.05, seed=5)
    for t in range(T):
        e = ref[t]
        assert g["k_star"][t] == e["k_star"], t
        assert (g["k_req"][t] == e["k_req"]).all(), t
        assert (g["num_accepted"][t] == e["num_accepted"]).all(), t
        assert (g["out_tokens"][t] == e["out_tokens"]).all(), t
        assert np.float64(g["alpha"][t]).tobytes() == np.float64(e["alpha"]).tobytes(), t
    assert (g["ctx_len"][-1] == rcl).all()
    assert (lp.ctx[T % 2].cpu().numpy() == rctx).all()


def test_alpha_shift_adaptation(loop_mod):
    # dataset shift: acceptance 0.9 -> 0.5 mid-run; the EWMA estimate reaches
    # within 0.05 of 0.5 in <= 100 steps and the chosen k drops
    B, L, V, K, T = 64, 256, 512, 5, 300
    at = [0.9] * 150 + [0.5] * 150
    lp, _, _ = _make(loop_mod, B, L, V, K, at, seed=9)
    lp.capture()
    lp.graph.replay()
    g = lp.logs()
    a = g["alpha"]
    assert abs(a[140:150].mean() - 0.9) < 0.05
    hit = next(t for t in range(150, T) if abs(a[t] - 0.5) < 0.05)
    assert hit - 150 <= 100, hit
    assert g["k_star"][200:].mean() < g["k_star"][100:150].mean()


def test_load_adaptation_disables_speculation(loop_mod):
    # PAPER.md:303 ("automatically disables speculative decoding" under load): with a
    # target whose cost grows with the batched tokens, the chosen k falls as the batch grows and
    # is 0 on > 90% of the steps at the largest batch (steps where some request has a proposal)
    heavy = (0.0, 0.5, 1.0)  # (ctx, batched, fixed) ms
    means, zero_frac = [], 0.0
    for B in (1, 4, 16, 64):
        lp, _, _ = _make(loop_mod, B, 256, 512, 5, [0.9] * 80, seed=13, alpha0=0.9, target=heavy)
        lp.capture()
        lp.graph.replay()
        g = lp.logs()
        has = g["proposal_len"].max(axis=1) > 0
        ks = g["k_star"][has]
        means.append(ks.mean())
        zero_frac = (ks == 0).mean()
    assert all(means[i] > means[i + 1] for i in range(3)), means
    assert zero_frac > 0.9, zero_frac


def test_estimator_world_consistency(loop_mod):
    # realised tokens per step match the estimator's sum_i l(alpha, k_i) within 5%
    B, L, V, K, T = 64, 256, 512, 5, 200
    lp, _, _ = _make(loop_mod, B, L, V, K, [0.8] * T, seed=17, alpha0=0.8)
    lp.capture()
    lp.graph.replay()
    g = lp.logs()
    real = (g["num_accepted"][50:] + 1).sum()
    pred = sum(oracle.expected_len(0.8, int(k)) for row in g["k_req"][50:] for k in row)
    assert abs(real / pred - 1) < 0.05, (real, pred)
