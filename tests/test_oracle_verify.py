"""Pins for the oracle's rejection-sampling verify (PAPER.md:18 [AD], 493-497 [BG]).

Each test checks the oracle against something that is not the oracle:
  * hand-computed tiny-vocabulary cases with injected uniforms (accept rule,
    residual, bonus, ties, one-hot drafts, q(x)=0 / p(x)=0, fallback);
  * the distribution laws that define speculative sampling: the first emitted
    token is distributed exactly as p ("zero accuracy loss"),
    P(m = j) follows the geometric chain whose mean is Eq. gen_len
    (PAPER.md:137), and at alpha = 0.7, k = 2 the case study's probabilities
    0.3 / 0.21 / 0.49 and expected latency 7.16 ms;
  * invariants: 0 <= m <= k, emitted prefix = drafts, exactly one
    bonus/correction token (min 1, max k+1 tokens).
"""
import numpy as np
import pytest
from scipy import stats

import oracle
import synth


def _one(p_rows, q_rows, drafts, k_max=None, u=None, E=None, vocab=None):
    p = np.asarray(p_rows, np.float32)
    q = None if q_rows is None else np.asarray(q_rows, np.float32)
    k = len(drafts)
    ro = np.array([0, k + 1], np.int32)
    return oracle.verify(p, q, ro, np.asarray(drafts, np.int32), np.array([7], np.uint32),
                         seed=1, step=0, k_max=k if k_max is None else k_max,
                         inj_u_acc=None if u is None else np.asarray(u, np.float32),
                         inj_E=None if E is None else np.asarray(E, np.float32), vocab=vocab)


P0 = [0.5, 0.25, 0.125, 0.125]
Q0 = [0.25, 0.5, 0.125, 0.125]
P1 = [0.1, 0.2, 0.3, 0.4]
ONES = [1.0, 1.0, 1.0, 1.0]


def test_accept_then_bonus():
    # x=1: u*q = 0.49*0.5 = 0.245 < p = 0.25 -> accept; bonus from p1, E = 1 -> argmax p1 = 3
    na, out, st = _one([P0, P1], [Q0], [1], u=[0.49], E=[ONES, ONES])
    assert st == 0 and na[0] == 1 and out[0].tolist() == [1, 3]


def test_reject_then_residual():
    # u = 0.5: 0.25 < 0.25 is false -> reject; residual max(0, p-q) = (.25, 0, 0, 0) -> 0 for any E
    for E1 in (ONES, [16.0, 1e-7, 1e-7, 1e-7]):
        na, out, st = _one([P0, P1], [Q0], [1], u=[0.5], E=[E1, ONES])
        assert st == 0 and na[0] == 0 and out[0].tolist() == [0, -1]


def test_race_picks_max_ratio():
    # bonus only (k = 0): scores w/E = (0.1, 0.2, 0.3, 4.0) -> 3 ; (10, .2, .3, .4) -> 0
    na, out, _ = _one([P1], None, [], E=[[1.0, 1.0, 1.0, 0.1]])
    assert na[0] == 0 and out[0].tolist() == [3]
    na, out, _ = _one([P1], None, [], E=[[0.01, 1.0, 1.0, 1.0]])
    assert out[0].tolist() == [0]


def test_race_tie_lowest_index():
    # equal scores at 1 and 2 -> lowest index 1
    na, out, _ = _one([[0.25] * 4], None, [], E=[[2.0, 1.0, 1.0, 2.0]])
    assert out[0].tolist() == [1]
    na, out, _ = _one([[0.25] * 4], None, [], E=[ONES])
    assert out[0].tolist() == [0]


def test_single_positive_weight():
    na, out, _ = _one([[0.0, 0.0, 1.0, 0.0]], None, [], E=[[1e-7, 1e-7, 16.0, 1e-7]])
    assert out[0].tolist() == [2]


def test_one_hot_drafts():
    # q one-hot at x=2: accept iff u < p(x) = 0.3 ; residual = p with x zeroed
    na, out, _ = _one([P1, P0], None, [2], u=[0.3], E=[ONES, ONES])
    assert na[0] == 0 and out[0].tolist() == [3, -1]
    na, out, _ = _one([P1, P0], None, [2], u=[0.3], E=[[1.0, 1.0, 1e-6, 1.0], ONES])
    assert out[0].tolist() == [3, -1]      # x itself has zero residual weight
    na, out, _ = _one([P1, P0], None, [2], u=[0.29], E=[ONES, ONES])
    assert na[0] == 1 and out[0].tolist() == [2, 0]


def test_q_zero_and_p_zero():
    # q(x) = 0 and p(x) > 0 -> accept for any u; p(x) = 0 -> reject even at u = 0
    p = [[0.1, 0.9, 0.0, 0.0], ONES]
    q = [[0.0, 0.5, 0.5, 0.0]]
    na, _, _ = _one(p, q, [0], u=[1.0 - 2 ** -24], E=[ONES, ONES])
    assert na[0] == 1
    na, out, _ = _one(p, q, [2], u=[0.0], E=[ONES, ONES])
    assert na[0] == 0 and out[0, 0] == 1   # residual (0.1, 0.4, 0, 0)/E=1 -> 1


def test_residual_all_zero_falls_back_to_p():
    # q >= p everywhere (unnormalised on purpose): reject, residual == 0 -> race over p_m
    p = [[0.1, 0.2, 0.3, 0.4], ONES]
    q = [[0.2, 0.2, 0.3, 0.4]]
    na, out, st = _one(p, q, [0], u=[0.6], E=[[1.0, 1.0, 1.0, 0.5], ONES])
    assert st == 0 and na[0] == 0 and out[0].tolist() == [3, -1]


def test_status_bad_token_bad_k_no_weight():
    na, out, st = _one([P0, P1], [Q0], [4], u=[0.1], E=[ONES, ONES])
    assert st & oracle.STATUS_BAD_TOKEN and na[0] == -1 and out[0].tolist() == [-1, -1]
    na, out, st = _one([P0, P1, P1], [Q0, Q0], [1, 1], k_max=1, u=[0.1, 0.1])
    assert st & oracle.STATUS_BAD_K and na[0] == -1
    na, out, st = _one([[0.0] * 4], None, [], E=[ONES])
    assert st & oracle.STATUS_NO_WEIGHT and out[0].tolist() == [-1]


def test_vocab_smaller_than_ld():
    # columns >= V are never read: put huge weight there
    p = np.array([[0.1, 0.2, 0.3, 0.4, 100.0, 100.0, 100.0, 100.0]], np.float32)
    na, out, _ = _one(p, None, [], E=[ONES + ONES], vocab=4)
    assert out[0].tolist() == [3]


def test_invariants_random_batch():
    vb = synth.make_verify_batch(B=64, V=96, k_max=8, lam=0.6, seed=5, ld=100)
    na, out, st = oracle.verify(vb.p.numpy(), vb.q.numpy(), vb.row_offsets.numpy(),
                                vb.draft_tokens.numpy(), vb.request_ids.numpy().view(np.uint32),
                                seed=99, step=3, k_max=8, vocab=96)
    assert st == 0
    ro = vb.row_offsets.numpy()
    d = vb.draft_tokens.numpy()
    for i in range(64):
        k = ro[i + 1] - ro[i] - 1
        m = na[i]
        assert 0 <= m <= k
        qb = ro[i] - i
        assert out[i, :m].tolist() == d[qb:qb + m].tolist()
        assert 0 <= out[i, m] < 96
        assert (out[i, m + 1:] == -1).all()


# ---------------------------------------------------------------------------
# distribution laws (the definition of speculative sampling)
# ---------------------------------------------------------------------------
PL = np.array([0.3, 0.2, 0.1, 0.1, 0.1, 0.1, 0.05, 0.05])
QL = np.array([0.1, 0.1, 0.2, 0.2, 0.1, 0.1, 0.1, 0.1])   # sum min(p, q) = 0.7


def _law_batch(N, k, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    p = np.tile(PL.astype(np.float32), (N * (k + 1), 1))
    q = np.tile(QL.astype(np.float32), (N * k, 1))
    drafts = rng.choice(8, size=N * k, p=QL).astype(np.int32)
    ro = np.arange(0, N * (k + 1) + 1, k + 1, dtype=np.int32)
    rid = np.arange(N, dtype=np.uint32)
    return p, q, ro, drafts, rid


@pytest.fixture(scope="module")
def law_k2():
    N = 200_000
    p, q, ro, d, rid = _law_batch(N, 2, seed=11)
    na, out, st = oracle.verify(p, q, ro, d, rid, seed=240614066, step=0, k_max=2)
    assert st == 0
    return na, out


def test_accepted_count_geometric_case_study(law_k2):
    na, _ = law_k2
    N = na.size
    alpha = float(np.minimum(PL, QL).sum())
    want = np.array([1 - alpha, alpha * (1 - alpha), alpha ** 2])   # 0.3, 0.21, 0.49
    np.testing.assert_allclose(want, [0.3, 0.21, 0.49], atol=1e-12)
    counts = np.bincount(na, minlength=3)
    chi = stats.chisquare(counts, want * N)
    assert chi.pvalue > 1e-4, (counts / N, chi)
    # expected per-token latency of the case study: 12.6 / 6.3 / 4.2 ms -> 7.16 ms
    lat = (counts / N * np.array([12.6, 6.3, 4.2])).sum()
    assert abs(lat - 7.16) < 0.03
    # Eq. gen_len: E[m+1] = l(alpha, k)
    assert abs((na + 1).mean() - oracle.expected_len(alpha, 2)) < 0.01


def test_first_token_distributed_as_p(law_k2):
    _, out = law_k2
    first = out[:, 0]
    counts = np.bincount(first, minlength=8)
    chi = stats.chisquare(counts, PL * first.size)
    assert chi.pvalue > 1e-4, (counts / first.size, chi)


def test_second_token_given_accept_distributed_as_p(law_k2):
    na, out = law_k2
    sel = out[na >= 1, 1]
    counts = np.bincount(sel, minlength=8)
    chi = stats.chisquare(counts, PL * sel.size)
    assert chi.pvalue > 1e-4, (counts / sel.size, chi)


def test_bonus_race_frequency_proportional_to_weight():
    # k = 0: the exponential race alone draws v with probability w_v / sum(w)
    N = 200_000
    w = np.array([1, 2, 3, 4, 5, 6, 7, 8], np.float32)
    p = np.tile(w, (N, 1))
    ro = np.arange(N + 1, dtype=np.int32)
    na, out, st = oracle.verify(p, None, ro, np.zeros(0, np.int32), np.arange(N, dtype=np.uint32),
                                seed=3, step=17, k_max=0)
    counts = np.bincount(out[:, 0], minlength=8)
    chi = stats.chisquare(counts, w.astype(np.float64) / float(w.sum()) * N)
    assert chi.pvalue > 1e-4, chi


def test_step_and_seed_change_draws():
    p, q, ro, d, rid = _law_batch(2000, 2, seed=1)
    a = oracle.verify(p, q, ro, d, rid, seed=5, step=0, k_max=2)[1]
    b = oracle.verify(p, q, ro, d, rid, seed=5, step=1, k_max=2)[1]
    c = oracle.verify(p, q, ro, d, rid, seed=6, step=0, k_max=2)[1]
    a2 = oracle.verify(p, q, ro, d, rid, seed=5, step=0, k_max=2)[1]
    assert (a == a2).all()
    assert (a != b).any() and (a != c).any()


def test_golden_case_study_values():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_worked_values.json")))
    cs = g["case_study"]
    a, k = cs["alpha"], cs["k"]
    probs = [a ** j * (1 - a) for j in range(k)] + [a ** k]
    np.testing.assert_allclose(probs, cs["prob_m"], atol=1e-12)
    lat = float(np.dot(probs, cs["per_token_latency_ms"]))
    assert abs(lat - cs["expected_latency_ms"]) < 0.005
    for a, k, want in g["expected_len"]["cases"]:
        assert abs(oracle.expected_len(a, k) - want) < 1e-12
    m = g["forward_time"]["model"]
    for c, b, want in g["forward_time"]["cases"]:
        assert abs(oracle.forward_time(m, c, b) - want) < 1e-12
