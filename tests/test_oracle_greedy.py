"""Pins for the greedy (temperature-0) verify oracle.

Greedy speculative decoding keeps draft j iff it equals the target's argmax at position j and
emits the target's argmax at the first mismatch (or after the last draft).  Pins: hand cases,
ties / NaN / negative values, numpy's first-occurrence argmax, and the temperature-0 limit of
the (separately pinned) sampling verify: with one-hot target rows at the argmax and one-hot
drafts, rejection sampling accepts exactly the argmax drafts and its residual / bonus race
returns the argmax, for every seed.
"""
import numpy as np

import oracle

S_BAD_TOKEN, S_BAD_K, S_NO_WEIGHT = oracle.STATUS_BAD_TOKEN, oracle.STATUS_BAD_K, oracle.STATUS_NO_WEIGHT


def _batch(rows_per_req, drafts_per_req):
    ks = [len(d) for d in drafts_per_req]
    p = np.concatenate([np.asarray(r, np.float32) for r in rows_per_req])
    ro = np.zeros(len(ks) + 1, np.int32)
    ro[1:] = np.cumsum(np.array(ks) + 1)
    d = np.array([x for ds in drafts_per_req for x in ds], np.int32)
    return p, ro, d


def test_hand_case_first_mismatch_and_correction():
    V = 5
    rows = np.zeros((4, V), np.float32)
    for j, a in enumerate([2, 4, 1, 0]):
        rows[j, a] = 0.6
        rows[j, (a + 1) % V] = 0.3
    p, ro, d = _batch([rows], [[2, 4, 3]])
    na, out, st = oracle.verify_greedy(p, ro, d, 3)
    assert na.tolist() == [2] and out.tolist() == [[2, 4, 1, -1]] and st == 0
    p, ro, d = _batch([rows], [[2, 4, 1]])  # all accepted -> bonus = argmax of row 3
    na, out, _ = oracle.verify_greedy(p, ro, d, 3)
    assert na.tolist() == [3] and out.tolist() == [[2, 4, 1, 0]]
    p, ro, d = _batch([rows], [[0, 4, 1]])  # first draft wrong -> m = 0, correction = 2
    na, out, _ = oracle.verify_greedy(p, ro, d, 3)
    assert na.tolist() == [0] and out.tolist() == [[2, -1, -1, -1]]


def test_ties_nan_negative_and_empty_rows():
    nan = np.nan
    cases = [
        ([0.25, 0.25, 0.25, 0.25], 0),          # all equal -> lowest index
        ([0.1, 0.4, 0.1, 0.4], 1),              # two maxima -> the first
        ([nan, 0.1, 0.5, nan], 2),              # NaN never selected
        ([-3.0, -1.0, -2.0, -1.0], 1),          # logits / negative values
        ([0.0, -0.0, 0.0, 0.0], 0),             # +0 == -0
        ([-np.inf, -np.inf, -5.0, np.inf], 3),
    ]
    for row, want in cases:
        p, ro, d = _batch([[row]], [[]])
        na, out, st = oracle.verify_greedy(p, ro, d, 0)
        assert na.tolist() == [0] and out[0, 0] == want and st == 0, row
    p, ro, d = _batch([[[nan, nan, nan]]], [[]])
    na, out, st = oracle.verify_greedy(p, ro, d, 0)
    assert out[0, 0] == -1 and st & S_NO_WEIGHT


def test_matches_numpy_argmax_and_invariants():
    rng = np.random.Generator(np.random.PCG64(31))
    for trial in range(200):
        B, V, K = int(rng.integers(1, 12)), int(rng.integers(1, 40)), int(rng.integers(0, 7))
        ks = rng.integers(0, K + 1, B)
        rows = [rng.integers(0, 4, (k + 1, V)).astype(np.float32) for k in ks]  # many ties
        drafts = []
        for r, k in zip(rows, ks):
            am = r.argmax(axis=1)
            ds = [int(am[j]) if rng.random() < 0.7 else int(rng.integers(0, V)) for j in range(k)]
            drafts.append(ds)
        p, ro, d = _batch(rows, drafts)
        na, out, st = oracle.verify_greedy(p, ro, d, K)
        assert st == 0
        for i in range(B):
            am = rows[i].argmax(axis=1)  # numpy: first occurrence of the maximum
            m = next((j for j in range(ks[i]) if drafts[i][j] != am[j]), ks[i])
            assert na[i] == m and 0 <= m <= ks[i]
            assert out[i, :m].tolist() == drafts[i][:m] and out[i, m] == am[m]
            assert (out[i, m + 1:] == -1).all()


def test_temperature_zero_limit_of_sampling_verify():
    # one-hot target rows at the argmax + one-hot drafts: the sampling verify (any seed) must
    # give exactly the greedy result on the original rows
    rng = np.random.Generator(np.random.PCG64(32))
    for trial in range(40):
        B, V, K = int(rng.integers(1, 10)), int(rng.integers(2, 64)), int(rng.integers(1, 6))
        ks = rng.integers(0, K + 1, B)
        rows = [rng.standard_normal((k + 1, V)).astype(np.float32) for k in ks]
        drafts = []
        for r, k in zip(rows, ks):
            am = r.argmax(axis=1)
            drafts.append([int(am[j]) if rng.random() < 0.75 else int(rng.integers(0, V)) for j in range(k)])
        p, ro, d = _batch(rows, drafts)
        gna, gout, _ = oracle.verify_greedy(p, ro, d, K)
        onehot = np.zeros_like(p)
        onehot[np.arange(p.shape[0]), p.argmax(axis=1)] = 1.0
        rid = np.arange(B, dtype=np.uint32)
        for seed in (1, 77, 2 ** 40 + 5):
            sna, sout, _ = oracle.verify(onehot, None, ro, d, rid, seed, trial, K)
            assert (sna == gna).all() and (sout == gout).all(), (trial, seed)


def test_bad_tokens_and_bad_k():
    rows = np.eye(4, dtype=np.float32)
    p, ro, d = _batch([rows[:3], rows[:2]], [[0, 1], [7]])
    na, out, st = oracle.verify_greedy(p, ro, d, 2)
    assert st & S_BAD_TOKEN and na.tolist() == [2, -1] and (out[1] == -1).all()
    p, ro, d = _batch([rows[:4]], [[0, 1, 2]])
    na, out, st = oracle.verify_greedy(p, ro, d, 2)  # k = 3 > k_max = 2
    assert st & S_BAD_K and (out == -1).all()
