"""GPU pins of the device RNG and E(u) against the oracle (exhaustive / KAT).

The race kernels evaluate E(u) with a log1p series near u = 1 and the double log
elsewhere; every one of the 2^23 race uniforms must give the oracle's (correctly
rounded) binary32 value.  The device Philox (generic and the row-specialised race
evaluation) must reproduce the Random123 KATs and the oracle on random counters.
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def tsv():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2406_14066_b200 import tsv as t
    return t


def test_race_E_exhaustive_matches_oracle(tsv):
    ref = oracle.E_table()
    got = tsv.tsv_debug_race_E(0, 1 << 23).cpu().numpy()
    bad = np.nonzero(got.view(np.uint32) != ref.view(np.uint32))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first m={bad[:5]}"


KATS = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
        ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
        ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
         (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]


@pytest.mark.parametrize("race_variant", [False, True])
def test_device_philox_kats_and_random(tsv, race_variant):
    for ctr, key, want in KATS:
        c = torch.tensor(np.array(ctr, np.uint32).view(np.int32), device="cuda")
        k = torch.tensor(np.array(key, np.uint32).view(np.int32), device="cuda")
        got = tsv.tsv_debug_philox(c, k, race_variant).cpu().numpy().view(np.uint32)
        assert [int(x) for x in got] == list(want)
    rng = np.random.Generator(np.random.PCG64(7))
    ctrs = rng.integers(0, 2 ** 32, (4096, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2 ** 32, 2, dtype=np.uint64).astype(np.uint32)
    got = tsv.tsv_debug_philox(torch.tensor(ctrs.reshape(-1).view(np.int32), device="cuda"),
                               torch.tensor(key.view(np.int32), device="cuda"), race_variant)
    got = got.cpu().numpy().view(np.uint32).reshape(-1, 4)
    for t in range(0, 4096, 97):
        assert (got[t] == oracle.philox4x32_10(ctrs[t], key)).all()


# ------------------------------------------------------------------ race logic with injected words
def _race_oracle(w, words):
    """Oracle token (k = 0 bonus row = w, injected E from the words) and its exact score bits."""
    E = _E_TABLE()[words & 0x7FFFFF]
    na, out, st = oracle.verify(w[None, :].astype(np.float32), None, np.array([0, 1], np.int32),
                                np.zeros(0, np.int32), np.zeros(1, np.uint32), 0, 0, 0,
                                inj_E=E[None, :].astype(np.float32))
    t = int(out[0, 0])
    score = np.float32(np.float32(w[t]) / E[t]).view(np.uint32) if t >= 0 else None
    return t, score


_EC = []


def _E_TABLE():
    if not _EC:
        _EC.append(oracle.E_table())
    return _EC[0]


def _gpu_race(tsv, w, words, prune=True):
    key = tsv.tsv_debug_race_row(torch.tensor(w, dtype=torch.float32, device=DEV),
                                 torch.tensor(words.view(np.int32), device=DEV), prune)
    if key == 0:
        return -1, None
    return 0xFFFFFFFF - (key & 0xFFFFFFFF), np.uint32(key >> 32)


def test_race_logic_with_adversarial_words(tsv):
    rng = np.random.Generator(np.random.PCG64(123))
    cases = []
    V = 1000
    cases.append((np.full(V, 0.001, np.float32), np.full(V, 0x12345678, np.uint32)))      # all tied -> index 0
    w = rng.random(V).astype(np.float32)
    x = rng.integers(0, 2 ** 32, V, dtype=np.uint64).astype(np.uint32)
    s = w / _E_TABLE()[x & 0x7FFFFF]
    top = int(np.argmax(s))
    w2, x2 = w.copy(), x.copy()
    w2[3], x2[3] = w[top], x[top]                                                         # exact tie at a lower index
    cases.append((w2, x2))
    cases.append((w, x))
    xe = x.copy()
    xe[::7] = 0x007FFFFF                                                                   # u -> 1: E tiny, scores huge
    xe[1::7] = 0                                                                           # u -> 2^-24: E large
    cases.append((w, xe))
    wz = w.copy()
    wz[rng.random(V) < 0.5] = 0.0
    wz[rng.random(V) < 0.2] = -1.0                                                         # non-positive: never win
    wz[rng.random(V) < 0.05] = np.nan
    cases.append((wz, x))
    cases.append((np.full(V, 1e-40, np.float32), x))                                      # denormal weights
    cases.append((np.zeros(V, np.float32), x))                                            # nothing positive
    big = (rng.zipf(1.2, 100003) * 1e-6).astype(np.float32)
    cases.append((big, rng.integers(0, 2 ** 32, 100003, dtype=np.uint64).astype(np.uint32)))
    for n, (w, x) in enumerate(cases):
        want_t, want_s = _race_oracle(w, x)
        for prune in (True, False):
            got_t, got_s = _gpu_race(tsv, w, x, prune)
            assert got_t == want_t, (n, prune, got_t, want_t)
            if want_t >= 0:
                assert got_s == want_s, (n, prune)
