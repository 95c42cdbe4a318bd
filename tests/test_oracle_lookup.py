"""Pins for the oracle's prompt-lookup proposal (Fig. PAPER.md:44-49).

Pinned against (a) hand-made contexts whose answers are worked out below,
(b) an independent numpy implementation (sliding windows + vectorised match),
which shares no loop structure with the oracle, on thousands of random small
contexts, and (c) the edge cases of reading R20 (L <= n, self-match excluded,
overlap allowed, truncation at the context end, no match -> length 0).
"""
import numpy as np
import pytest

import oracle
import synth
from numpy.lib.stride_tricks import sliding_window_view


def numpy_lookup(c, n_min, n_max, K):
    c = np.asarray(c, np.int64)
    L = c.size
    for n in range(n_max, n_min - 1, -1):
        if L < n + 1:
            continue
        win = sliding_window_view(c[:L - 1], n)          # win[s] = c[s:s+n], s <= L-n-1
        hits = np.nonzero((win == c[L - n:]).all(axis=1))[0]
        if hits.size:
            s = int(hits.max())
            return c[s + n: min(s + n + K, L)].tolist()
    return []


def run(ctxs, n_min, n_max, K):
    offs = np.zeros(len(ctxs) + 1, np.int32)
    offs[1:] = np.cumsum([len(c) for c in ctxs])
    flat = np.concatenate([np.asarray(c, np.int32) for c in ctxs]) if ctxs else np.zeros(0, np.int32)
    props, plen = oracle.lookup(flat, offs, n_min, n_max, K)
    return [props[i, :plen[i]].tolist() for i in range(len(ctxs))], props, plen


def test_hand_cases():
    # "a b c d a b" with n=2: trailing "a b" matches at s=0 -> propose "c d a b"[:K]
    got, props, plen = run([[1, 2, 3, 4, 1, 2]], 2, 2, 3)
    assert got == [[3, 4, 1]] and props[0].tolist() == [3, 4, 1]
    # latest match wins: "x y 5 x y 6 x y" -> s=3 (latest), propose "6 x y"
    got, _, _ = run([[7, 8, 5, 7, 8, 6, 7, 8]], 2, 2, 5)
    assert got == [[6, 7, 8]]
    # longest n first: n=3 matches "1 2 3" at s=0 although n=1 matches "3" later
    got, _, _ = run([[1, 2, 3, 9, 3, 4, 1, 2, 3]], 1, 3, 2)
    assert got == [[9, 3]]
    # no repeats -> nothing (request R2 of Fig. PAPER.md:44-49), padded with -1
    got, props, plen = run([[1, 2, 3, 4, 5]], 1, 3, 4)
    assert got == [[]] and plen[0] == 0 and (props[0] == -1).all()
    # match at s = L-n-1 gives a 1-token proposal (the last token)
    got, _, _ = run([[5, 6, 1, 1]], 1, 1, 5)
    assert got == [[1]]
    # all-same tokens: overlap allowed, latest start s = L-n-1
    got, _, _ = run([[4] * 10], 3, 3, 5)
    assert got == [[4]]
    # truncation: proposal cut at the context end
    got, _, _ = run([[1, 2, 3, 1, 2]], 2, 2, 10)
    assert got == [[3, 1, 2]]


@pytest.mark.parametrize("L", [0, 1, 2, 3, 4, 5])
def test_short_contexts(L):
    ctx = list(range(L)) if L < 3 else [1] * L
    got, _, plen = run([ctx], 1, 4, 5)
    assert got[0] == numpy_lookup(ctx, 1, 4, 5)
    if L <= 1:
        assert plen[0] == 0


def test_against_independent_numpy_random():
    rng = np.random.Generator(np.random.PCG64(20240614))
    ctxs, params = [], []
    for trial in range(3000):
        L = int(rng.integers(0, 41))
        A = int(rng.integers(1, 5))
        ctxs.append(rng.integers(0, A, L).astype(np.int32))
    for n_min, n_max, K in [(1, 1, 1), (1, 4, 5), (2, 3, 3), (3, 3, 5), (4, 4, 2), (1, 8, 7)]:
        got, _, _ = run(ctxs, n_min, n_max, K)
        for c, g in zip(ctxs, got):
            assert g == numpy_lookup(c, n_min, n_max, K), (c.tolist(), n_min, n_max, K)


def test_synthetic_pld_contexts_have_matches():
    ctx, offs = synth.make_contexts(B=16, L=512, seed=3)
    props, plen = oracle.lookup(ctx, offs, 3, 3, 5)
    for i in range(16):
        c = ctx[offs[i]:offs[i + 1]]
        assert props[i, :plen[i]].tolist() == numpy_lookup(c, 3, 3, 5)
    assert (plen > 0).any()
