"""Pins for the oracle's goodput adaptor (PAPER.md:97-143, 256-270 [AD]) and alpha update.

Against: Eq. gen_len's closed form and the SPEC.md worked values
(2.19, 2.7731, l(0,k)=1, l(1,k)=k+1); Eq. forward-time worked examples
(SPEC.md:59-60); the batch-latency example under the paper's product form
T_draft = s * T_fwd; the search's exhaustiveness and strict
'>' tie rule (Listing 2); the paper's qualitative insights 1-2
 and alpha = 0 -> no speculation; power-of-two scale
invariance; the OOM skip; the moving-average worked examples
and convergence bound.
"""
import math

import numpy as np
import pytest

import oracle
import synth

T = synth.SPEC_DESK_TARGET
D = synth.SPEC_DESK_DRAFT


@pytest.mark.parametrize("a,k,want", [(0.7, 2, 2.19), (0.7, 4, 2.7731), (0.0, 5, 1.0),
                                      (1.0, 3, 4.0), (0.5, 0, 1.0), (1.0, 0, 1.0)])
def test_expected_len_worked_values(a, k, want):
    assert abs(oracle.expected_len(a, k) - want) < 1e-12


def test_expected_len_closed_form():
    for a in np.linspace(0.0, 0.99, 34):
        for k in range(16):
            closed = (1 - a ** (k + 1)) / (1 - a)
            assert abs(oracle.expected_len(a, k) - closed) < 1e-12
    # Horner reaches the a=1 limit exactly (k+1) where the closed form divides by zero
    for k in range(16):
        assert oracle.expected_len(1.0, k) == k + 1


def test_forward_time_worked():
    assert oracle.forward_time(T, 0, 0) == 2.0
    assert abs(oracle.forward_time(T, 1000, 100) - 8.0) < 1e-12
    assert abs(oracle.forward_time(T, 1000, 200) - oracle.forward_time(T, 1000, 100) - 5.0) < 1e-12


def test_batch_latency_product_form():
    # B=1, context 100, k=2 draft: T_target = .001*100 + .05*3 + 2 = 2.25,
    # T_draft = 2 * (.0001*100 + .005*1 + .2) = 0.43  ->  2.68 ms (product form)
    a = 0.7
    _, g = oracle.choose_k(a, [100], [8], 8, oracle.POLICY_DRAFT, T, D)
    assert abs(oracle.expected_len(a, 2) / g[2] - 2.68) < 1e-8   # token sums are 2^-32 fixed point
    # k = 0: target only with 1 batched token per request (goodput reduces to throughput)
    assert abs(1.0 / g[0] - (0.1 + 0.05 + 2.0)) < 1e-8


def test_two_request_accept_len():
    # batch of 2, alpha 0.7, k=2 -> accepted length 4.38
    _, g = oracle.choose_k(0.7, [100, 100], [8, 8], 8, oracle.POLICY_DRAFT, T, D)
    lat = oracle.forward_time(T, 200, 6) + 2 * oracle.forward_time(D, 200, 2)
    assert abs(g[2] * lat - 4.38) < 1e-8


def test_exhaustive_strict_argmax():
    rng = np.random.Generator(np.random.PCG64(1))
    for trial in range(200):
        B = int(rng.integers(1, 40))
        ctx, cap = synth.make_goodput_instance(B, 8, seed=trial)
        a = float(rng.uniform(0.0, 1.0))
        k, g = oracle.choose_k(a, ctx, cap, 8, oracle.POLICY_DRAFT, T, D)
        assert g[k] == g.max()
        assert k == int(np.argmax(g))   # first maximum = smaller k on ties


def test_alpha_zero_disables_and_pld_extremes():
    ctx = np.full(8, 256, np.int32)
    k, _ = oracle.choose_k(0.0, ctx, np.full(8, 8, np.int32), 8, oracle.POLICY_DRAFT, T, D)
    assert k == 0
    caps = np.array([5, 0, 5, 3, 5, 0, 5, 5], np.int32)
    v, _ = oracle.choose_k(0.0, ctx, caps, 5, oracle.POLICY_PLD, T, D, pld_cost_ms=0.05)
    assert v == 0
    v, _ = oracle.choose_k(1.0, ctx, caps, 5, oracle.POLICY_PLD, T, D, pld_cost_ms=0.05)
    assert v == 5


def test_insight_1_small_batch_longer_k():
    # PAPER.md:88 "small batch -> longer k" at alpha .9, ctx 256/request
    ks = []
    for B in (1, 4, 16, 64):
        k, _ = oracle.choose_k(0.9, np.full(B, 256, np.int32), np.full(B, 8, np.int32), 8,
                               oracle.POLICY_DRAFT, T, D)
        ks.append(k)
    assert all(a >= b for a, b in zip(ks, ks[1:])) and ks[0] > ks[-1], ks


def test_insight_2_accurate_longer_k():
    # PAPER.md:91 "propose more for accurate batches" at batch 8
    ks = []
    for a in (0.3, 0.5, 0.7, 0.9):
        k, _ = oracle.choose_k(a, np.full(8, 256, np.int32), np.full(8, 8, np.int32), 8,
                               oracle.POLICY_DRAFT, T, D)
        ks.append(k)
    assert all(x <= y for x, y in zip(ks, ks[1:])) and ks[0] < ks[-1], ks


def test_scale_invariance_power_of_two():
    rng = np.random.Generator(np.random.PCG64(9))
    for trial in range(100):
        B = int(rng.integers(1, 64))
        ctx, cap = synth.make_goodput_instance(B, 8, seed=100 + trial)
        a = float(rng.uniform(0.2, 0.95))
        k1, _ = oracle.choose_k(a, ctx, cap, 8, oracle.POLICY_DRAFT, T, D)
        k2, _ = oracle.choose_k(a, ctx, cap, 8, oracle.POLICY_DRAFT,
                                [4 * x for x in T], [4 * x for x in D])
        assert k1 == k2


def test_oom_skip():
    ctx = np.full(4, 100, np.int32)
    cap = np.full(4, 8, np.int32)
    k_free, g = oracle.choose_k(0.95, ctx, cap, 8, oracle.POLICY_DRAFT, T, D, kv_free_slots=-1)
    assert k_free > 2
    # only k with 4*(k+1) <= 12 fit -> k <= 2
    k_lim, g = oracle.choose_k(0.95, ctx, cap, 8, oracle.POLICY_DRAFT, T, D, kv_free_slots=12)
    assert k_lim <= 2 and all(g[k] == -1.0 for k in range(3, 9))


def test_per_request_alpha_and_caps():
    # per-request alpha equal to the global one gives the same answer
    ctx, cap = synth.make_goodput_instance(33, 8, seed=4)
    k1, g1 = oracle.choose_k(0.8, ctx, cap, 8, oracle.POLICY_DRAFT, T, D)
    k2, g2 = oracle.choose_k(np.full(33, 0.8), ctx, cap, 8, oracle.POLICY_DRAFT, T, D)
    assert k1 == k2 and (g1 == g2).all()
    # token sum uses k_i = min(k, cap_i): with caps all 0 the goodput is flat in k for PLD
    _, g = oracle.choose_k(0.8, ctx, np.zeros(33, np.int32), 5, oracle.POLICY_PLD, T, D,
                           pld_cost_ms=0.05)
    assert np.all(g == g[0])


# ---------------------------------------------------------------------------
# acceptance update (Listing 1 UpdateGlobalAcceptance)
# ---------------------------------------------------------------------------
def _ro(ks):
    ro = np.zeros(len(ks) + 1, np.int32)
    ro[1:] = np.cumsum(np.asarray(ks) + 1)
    return ro


def test_update_worked_examples():
    # rate .5 step .5 -> .5 ; rate .5 step 1.0 -> .55
    assert abs(oracle.update(0.5, [1, 1], _ro([2, 2]), estimator=oracle.EST_PROPOSED) - 0.5) < 1e-15
    assert abs(oracle.update(0.5, [2, 2], _ro([2, 2]), estimator=oracle.EST_PROPOSED) - 0.55) < 1e-15
    # TESTED estimator: m=1 of k=2 tested 2 positions (one accept + one reject) -> r = .5
    assert abs(oracle.update(0.5, [1, 2], _ro([2, 2])) - (0.9 * 0.5 + 0.1 * (3 / 4))) < 1e-15


def test_update_nothing_tested_keeps_alpha():
    assert oracle.update(0.42, [0, 0], _ro([0, 0])) == 0.42


def test_update_convergence_bound():
    # repeated step rate 0.8 converges within 1e-3 after <= 66 updates
    for a0 in (0.0, 0.3, 1.0):
        a = a0
        for _ in range(66):
            a = oracle.update(a, [4], _ro([5]), estimator=oracle.EST_PROPOSED)
        assert abs(a - 0.8) < 1e-3


def test_update_per_request():
    a = oracle.update(np.array([0.5, 0.5, 0.9]), [2, 0, 0], _ro([2, 3, 0]))
    np.testing.assert_allclose(a, [0.55, 0.45, 0.9], atol=1e-15)


def test_tested_estimator_is_unbiased_for_geometric_chain():
    # Monte Carlo: m ~ truncated geometric(alpha) with ragged k; sum m / sum tested -> alpha
    rng = np.random.Generator(np.random.PCG64(5))
    alpha, N = 0.7, 400_000
    ks = rng.integers(0, 9, N)
    fails = rng.geometric(1 - alpha, N) - 1   # number of successes before the first failure
    m = np.minimum(fails, ks)
    r_tested = m.sum() / (m + (m < ks)).sum()
    assert abs(r_tested - alpha) < 0.005
    r_prop = m.sum() / ks.sum()
    assert r_prop < alpha - 0.1   # SPEC's per-proposed estimator is biased low (reading R18)
    got = oracle.update(0.0, m.astype(np.int32), _ro(ks), decay=0.0)
    assert abs(got - r_tested) < 1e-12
