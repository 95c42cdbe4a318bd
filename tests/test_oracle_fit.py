"""Pins for the latency-model fit oracle (reading R25; PAPER.md:106-113 Eq. forward-time,
SPEC.md:44-52): OLS on (context, batched, 1) with clamp-and-refit of negative coefficients."""
import numpy as np
import pytest

import oracle

PLANT = (0.001, 0.05, 2.0)  # SPEC desk target profile


def _grid():
    c, b = np.meshgrid(np.array([100, 400, 900, 1600, 2500.0]), np.array([1, 8, 32, 64, 128.0]))
    return c.ravel(), b.ravel()


def test_planted_recovery_noiseless():
    c, b = _grid()
    t = PLANT[0] * c + PLANT[1] * b + PLANT[2]
    coef, r2 = oracle.fit_latency(c, b, t)
    assert np.allclose(coef, PLANT, rtol=0, atol=1e-9) and r2 == pytest.approx(1.0, abs=1e-12)
    pred = coef[0] * c + coef[1] * b + coef[2]
    assert np.abs(pred - t).max() < 1e-9  # fit -> predict round trip


def test_constant_function():
    c, b = _grid()
    coef, r2 = oracle.fit_latency(c, b, np.full(c.size, 3.0))
    assert np.allclose(coef, (0.0, 0.0, 3.0), atol=1e-12) and r2 == 1.0


def test_noise_recovery_within_5_percent():
    rng = np.random.Generator(np.random.PCG64(61))
    c = rng.integers(100, 4096, 200).astype(np.float64)
    b = rng.integers(1, 256, 200).astype(np.float64)
    t = PLANT[0] * c + PLANT[1] * b + PLANT[2] + rng.normal(0, 0.01, 200)
    coef, r2 = oracle.fit_latency(c, b, t)
    assert np.all(np.abs(np.array(coef) - PLANT) / PLANT < 0.05) and r2 > 0.999


def test_unclamped_matches_numpy_lstsq():
    rng = np.random.Generator(np.random.PCG64(62))
    for trial in range(50):
        n = int(rng.integers(3, 60))
        c = rng.uniform(0, 5000, n)
        b = rng.uniform(0, 300, n)
        t = rng.uniform(0.5, 2, 3) @ np.vstack([c / 1000, b / 100, np.ones(n)]) + rng.normal(0, 0.05, n)
        ref, *_ = np.linalg.lstsq(np.column_stack([c, b, np.ones(n)]), t, rcond=None)
        if (ref < 0).any():
            continue
        coef, _ = oracle.fit_latency(c, b, t)
        assert np.allclose(coef, ref, rtol=1e-8, atol=1e-12), trial


def test_negative_coefficient_clamped_and_refit():
    rng = np.random.Generator(np.random.PCG64(63))
    c = rng.uniform(100, 4000, 80)
    b = rng.uniform(1, 200, 80)
    t = -0.0005 * c + 0.05 * b + 6.0 + rng.normal(0, 0.01, 80)  # planted negative context slope
    coef, _ = oracle.fit_latency(c, b, t)
    assert coef[0] == 0.0 and min(coef) >= 0.0
    ref, *_ = np.linalg.lstsq(np.column_stack([b, np.ones(80)]), t, rcond=None)  # refit on the free columns
    assert np.allclose(coef[1:], ref, rtol=1e-9)


def test_errors():
    with pytest.raises(ValueError, match="TooFewSamples"):
        oracle.fit_latency([1, 2], [3, 4], [5, 6])
    c = np.arange(10.0)
    with pytest.raises(ValueError, match="DegenerateDesign"):
        oracle.fit_latency(c, 2 * c, 3 * c + 1)
