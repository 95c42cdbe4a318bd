"""Pins for the softmax-from-logits oracle (reading R23).

p = RN32(expf(RN32(RN32(z - M) * RN32(1/tau))) * RN32(1/S)), S the binary64 sum of the fp32
exponentials.  Checked against float64 softmax (scipy) to 1e-6 relative, closed forms (uniform
logits -> RN32(1/V), a dominant logit -> one-hot), exact shift invariance on a dyadic grid, the
temperature law softmax(z / tau) and normalisation.
"""
import numpy as np
from scipy.special import softmax

import oracle


def test_matches_float64_softmax():
    rng = np.random.Generator(np.random.PCG64(41))
    for V, tau, sigma in [(32000, 1.0, 3.0), (4099, 0.7, 2.0), (13, 1.5, 8.0), (1, 1.0, 1.0)]:
        z = (rng.standard_normal((6, V)) * sigma).astype(np.float32)
        p = oracle.softmax_rows(z, tau)
        ref = softmax(z.astype(np.float64) / np.float64(np.float32(tau)), axis=1)
        # fp32 argument a = (z - M) / tau carries half an ulp: exp turns that into a relative
        # error of |a| 2^-24; plus a few ulps from expf, 1/S and the product
        a = np.abs(z.astype(np.float64) - z.max(axis=1, keepdims=True)) / tau
        bound = (a + 4.0) * 2.0 ** -23
        big = ref > 1e-30
        rel = np.abs(p[big] - ref[big]) / ref[big]
        assert (rel <= bound[big]).all(), (V, tau, (rel / bound[big]).max())
        assert rel[a[big] < 4].max() < 1e-6  # the bulk of the mass: within 1e-6
        assert np.abs(p.astype(np.float64).sum(axis=1) - 1).max() < 1e-6 * max(1, V / 1000)


def test_closed_forms():
    for V in (1, 3, 100, 32000):
        p = oracle.softmax_rows(np.zeros((1, V), np.float32))
        assert (p == np.float32(1.0 / V)).all()
    z = np.full((1, 50), -200.0, np.float32)
    z[0, 17] = 0.0
    p = oracle.softmax_rows(z)
    assert p[0, 17] == 1.0 and (np.delete(p[0], 17) == 0).all()


def test_shift_invariance_exact_on_dyadic_grid():
    rng = np.random.Generator(np.random.PCG64(42))
    z = (rng.integers(-64, 64, (4, 257)) / 8.0).astype(np.float32)  # multiples of 1/8: z - M exact
    for c in (1.0, -37.5, 1024.0):
        assert (oracle.softmax_rows(z + np.float32(c)) == oracle.softmax_rows(z)).all()


def test_temperature_law():
    rng = np.random.Generator(np.random.PCG64(43))
    z = (rng.standard_normal((3, 1000)) * 2).astype(np.float32)
    for tau in (0.5, 2.0, 4.0):  # 1/tau exact: softmax(z, tau) == softmax(z * (1/tau), 1) bit for bit
        assert (oracle.softmax_rows(z, tau) == oracle.softmax_rows(z * np.float32(1.0 / tau), 1.0)).all()


def test_padding_columns_zeroed_and_vocab_respected():
    z = np.zeros((2, 12), np.float32)
    z[:, 10:] = 50.0  # beyond vocab: ignored
    p = oracle.softmax_rows(z, 1.0, vocab=10)
    assert (p[:, :10] == np.float32(0.1)).all() and (p[:, 10:] == 0).all()
