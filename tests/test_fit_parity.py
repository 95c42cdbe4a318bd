"""libtsv's host latency-model fit (Householder QR) vs the oracle (normal equations): same
definition (reading R25), different algorithms -> agreement within 1e-9 relative.  Host-only
code: runs without a GPU."""
import numpy as np
import pytest

import oracle


@pytest.fixture(scope="module")
def tsv():
    from paper_2406_14066_b200 import tsv as t
    return t


def test_fit_matches_oracle(tsv):
    rng = np.random.Generator(np.random.PCG64(71))
    for trial in range(200):
        n = int(rng.integers(3, 120))
        c = rng.integers(0, 8192, n).astype(np.float64)
        b = rng.integers(1, 512, n).astype(np.float64)
        plant = rng.uniform(-0.002, 0.004, 3) * np.array([1, 20, 1000])  # some negative -> clamping
        t = plant[0] * c + plant[1] * b + plant[2] + rng.normal(0, 0.02, n)
        try:
            want, wr2 = oracle.fit_latency(c, b, t)
        except ValueError:
            continue
        got, gr2 = tsv.tsv_fit_latency_model(c, b, t)
        assert np.allclose(got, want, rtol=1e-9, atol=1e-12), (trial, got, want)
        assert gr2 == pytest.approx(wr2, rel=1e-9, abs=1e-12)
        assert min(got) >= 0.0


def test_fit_planted_and_errors(tsv):
    c, b = np.meshgrid(np.array([100, 400, 900, 1600, 2500.0]), np.array([1, 8, 32, 64, 128.0]))
    c, b = c.ravel(), b.ravel()
    got, r2 = tsv.tsv_fit_latency_model(c, b, 0.001 * c + 0.05 * b + 2.0)
    assert np.allclose(got, (0.001, 0.05, 2.0), atol=1e-9) and r2 == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(tsv.TsvError):
        tsv.tsv_fit_latency_model([1.0, 2.0], [1.0, 2.0], [1.0, 2.0])
    x = np.arange(10.0)
    with pytest.raises(tsv.TsvError):
        tsv.tsv_fit_latency_model(x, 2 * x, 3 * x + 1)
