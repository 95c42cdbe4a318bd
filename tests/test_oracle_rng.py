"""Pins for the oracle's Philox4x32-10, uniform conversions and E(u) (R2, R6, R9).

Philox: Random123 known-answer vectors (kat_vectors, philox4x32_10), which
fix every multiplier, Weyl increment, round count and word order.
Uniforms: boundary words whose values follow from the definitions by hand.
E(u): exhaustive over all 2^23 race uniforms against the correctly rounded
binary32 value of -ln(u), established independently with numpy's float64 log
plus a check that no value lies within 8 float64 ulps of a binary32 midpoint.
"""
import numpy as np
import pytest

import oracle

KATS = [
    # (counter, key, expected) -- Random123 philox4x32_10 known-answer tests
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KATS)
def test_philox_kat(ctr, key, want):
    got = oracle.philox4x32_10(ctr, key)
    assert [int(x) for x in got] == list(want)


def test_u_acc_boundaries():
    # u_acc = (x >> 8) * 2^-24 on [0, 1)
    assert oracle.u_acc(0) == 0.0
    assert oracle.u_acc(255) == 0.0
    assert oracle.u_acc(256) == 2.0 ** -24
    assert oracle.u_acc(0xFFFFFFFF) == 1.0 - 2.0 ** -24
    assert oracle.u_acc(0x80000000) == 0.5


def test_u_race_boundaries():
    # u_race = (2 (x & 0x7FFFFF) + 1) 2^-24 in (0, 1): never 0 or 1; high 9 bits ignored
    assert oracle.u_race(0) == 2.0 ** -24
    assert oracle.u_race(0xFF800000) == 2.0 ** -24
    assert oracle.u_race(1) == 3 * 2.0 ** -24
    assert oracle.u_race(0x7FFFFF) == 1.0 - 2.0 ** -24
    assert oracle.u_race(0xFFFFFFFF) == 1.0 - 2.0 ** -24
    assert oracle.u_race(0x400000) == 0.5 + 2.0 ** -24


def _correctly_rounded_neg_log():
    m = np.arange(1 << 23, dtype=np.float64)
    u = (2.0 * m + 1.0) * 2.0 ** -24           # exact in float64
    l = -np.log(u)                               # float64, error <= 1-2 ulp
    e = l.astype(np.float32)
    # distance (in float64 ulps of l) from l to the nearest binary32 rounding midpoint
    e64 = e.astype(np.float64)
    up = np.nextafter(e, np.float32(np.inf)).astype(np.float64)
    dn = np.nextafter(e, np.float32(0)).astype(np.float64)
    mid_up = (e64 + up) / 2.0
    mid_dn = (e64 + dn) / 2.0
    ulp = np.spacing(l)
    dist = np.minimum(np.abs(l - mid_up), np.abs(l - mid_dn)) / ulp
    return u, e, dist


def test_E_exhaustive_correctly_rounded():
    u, ref, dist = _correctly_rounded_neg_log()
    # every rounding is unambiguous: float64 log (error <= 2 ulp) lies >= 8 ulp from
    # any binary32 midpoint, so float32(float64 log) IS the correctly rounded -ln(u)
    assert float(dist.min()) > 8.0, float(dist.min())
    got = oracle.E_table()
    assert got.dtype == np.float32
    mism = np.nonzero(got.view(np.uint32) != ref.view(np.uint32))[0]
    assert mism.size == 0, f"{mism.size} E(u) values not correctly rounded, first at m={mism[:5]}"
    # E > 0 everywhere and bounded: [5.96e-8, 16.64]
    assert float(got.min()) > 5.9e-8 and float(got.max()) < 16.7


def test_E_scalar_matches_table():
    tab = oracle.E_table()
    for m in (0, 1, 12345, (1 << 22), (1 << 23) - 1):
        u = (2 * m + 1) * 2.0 ** -24
        assert np.float32(oracle.E(u)) == tab[m]
