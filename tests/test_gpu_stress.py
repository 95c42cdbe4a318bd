"""Randomised parity (a bounded slice of scripts/stress_parity.py): random batch shapes, vocab sizes
(ragged included), chunk widths, dense / one-hot q, prune on / off for the verify, and tie-heavy rows for
the greedy verify -- every output bit-exact against the oracle.  Fixed seeds, so a failure reproduces."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def tsv():
    from paper_2406_14066_b200 import tsv as t
    return t


def _np(t):
    return None if t is None else t.detach().cpu().numpy()


@pytest.mark.parametrize("seed", [101, 202, 303])
def test_random_verify_parity(tsv, seed):
    rng = np.random.default_rng(seed)
    for _ in range(40):
        B = int(rng.integers(1, 96))
        V = int(rng.choice([int(rng.integers(1, 600)), int(rng.integers(600, 20000)), 32000]))
        k_max = int(rng.integers(0, 9))
        dense = bool(rng.integers(0, 2))
        chunk = int(rng.choice([0, 128, 384, 1792]))
        flags = tsv.VERIFY_NO_PRUNE if rng.random() < 0.2 else 0
        s, step = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**32))
        vb = synth.make_verify_batch(B=B, V=V, k_max=k_max, lam=float(rng.uniform(0.05, 0.98)),
                                     seed=int(rng.integers(0, 2**31)), dense_q=dense)
        ona, oout, ost = oracle.verify(_np(vb.p), _np(vb.q), _np(vb.row_offsets), _np(vb.draft_tokens),
                                       _np(vb.request_ids).view(np.uint32), s, step, k_max, vocab=V)
        g = vb.to(DEV)
        st = torch.zeros(1, dtype=torch.int32, device=DEV)
        na, out = tsv.tsv_verify_accept(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, s, step, k_max,
                                        device_status=st, vocab=V, chunk=chunk, flags=flags)
        torch.cuda.synchronize()
        case = dict(B=B, V=V, k_max=k_max, dense=dense, chunk=chunk, flags=flags, seed=s, step=step)
        assert (_np(na) == ona).all() and (_np(out) == oout).all(), case
        assert int(st.item()) == ost, case


@pytest.mark.parametrize("seed", [404, 505])
def test_random_greedy_parity(tsv, seed):
    rng = np.random.default_rng(seed)
    for _ in range(60):
        B = int(rng.integers(1, 96))
        V = int(rng.choice([int(rng.integers(1, 600)), int(rng.integers(600, 20000)), 32000]))
        k_max = int(rng.integers(0, 9))
        chunk = int(rng.choice([0, 128, 640]))
        ks = rng.integers(0, k_max + 1, B)
        ro = np.zeros(B + 1, np.int32)
        ro[1:] = np.cumsum(ks + 1)
        ld = (V + 3) // 4 * 4
        ties = rng.random() < 0.5
        p = (rng.integers(0, 5, (int(ro[-1]), ld)) if ties else rng.standard_normal((int(ro[-1]), ld))).astype(np.float32)
        am = p[:, :V].argmax(axis=1)
        drafts = np.array([int(am[ro[i] + j]) if rng.random() < 0.7 else int(rng.integers(0, V))
                           for i in range(B) for j in range(ks[i])], np.int32)
        ona, oout, ost = oracle.verify_greedy(p, ro, drafts, k_max, vocab=V)
        st = torch.zeros(1, dtype=torch.int32, device=DEV)
        dt = torch.tensor(drafts if len(drafts) else np.zeros(0, np.int32), dtype=torch.int32, device=DEV)
        na, out = tsv.tsv_verify_greedy(torch.tensor(p, device=DEV), torch.tensor(ro, device=DEV), dt, k_max,
                                        device_status=st, vocab=V, chunk=chunk)
        torch.cuda.synchronize()
        case = dict(B=B, V=V, k_max=k_max, ties=ties, chunk=chunk)
        assert (_np(na) == ona).all() and (_np(out) == oout).all(), case
        assert int(st.item()) == ost, case
