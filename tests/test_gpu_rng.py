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
