/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the TurboSpec
 * propose / verify / accept step (arXiv 2406.14066), written from the paper
 * and the readings listed in DESIGN.md section 3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load this library.  It shares no code, header,
 * constant table or helper with the CUDA path in paper_2406_14066_b200/ and
 * neither side includes or imports the other.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared (no FMA
 * contraction, IEEE binary32/binary64 on SSE, denormals honoured).
 *
 * Every floating-point decision below is taken in the precision the CUDA
 * path takes it in (binary32 for probabilities and race scores, binary64
 * for the goodput model), because a floating-point result decides an integer
 * (accept/reject, argmax) and both sides must decide it identically.
 *
 * Pins: tests/test_oracle_*.py check every function here against something
 * that is not this code (KATs, closed forms, worked examples from the paper,
 * brute force, distribution laws).  Functions with no such pin: none; the
 * counter layout and uniform conversions are design choices (R6)
 * pinned by their own boundary values.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3").  The paper names no RNG (reading R6); we
 * use the standard 10-round Philox4x32 with its published multipliers and
 * Weyl key increments.                                                      */
/* ------------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    int round;
    for (round = 0; round < 10; ++round) {
        uint64_t prod0, prod1;
        uint32_t hi0, lo0, hi1, lo1;
        if (round > 0) { /* key schedule: bump between rounds */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        hi0 = (uint32_t)(prod0 >> 32); lo0 = (uint32_t)prod0;
        hi1 = (uint32_t)(prod1 >> 32); lo1 = (uint32_t)prod1;
        {
            uint32_t n0 = hi1 ^ c1 ^ k0;
            uint32_t n1 = lo1;
            uint32_t n2 = hi0 ^ c3 ^ k1;
            uint32_t n3 = lo0;
            c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Counter layout (R6): c0 = quad index (vocab index >> 2, 0 for
 * acceptance draws), c1 = (purpose << 16) | position, c2 = global request id,
 * c3 = step.  Key = (seed low 32 bits, seed high 32 bits).                  */
static uint32_t philox_word(uint64_t seed, uint32_t quad, uint32_t purpose, uint32_t position,
                            uint32_t request_id, uint32_t step, uint32_t word)
{
    uint32_t ctr[4], key[2], out[4];
    ctr[0] = quad;
    ctr[1] = (purpose << 16) | (position & 0xFFFFu);
    ctr[2] = request_id;
    ctr[3] = step;
    key[0] = (uint32_t)(seed & 0xFFFFFFFFu);
    key[1] = (uint32_t)(seed >> 32);
    oracle_philox4x32_10(ctr, key, out);
    return out[word];
}

/* Acceptance uniform on the 2^-24 grid in [0, 1) (R2). */
float oracle_u_acc(uint32_t x)
{
    return (float)(x >> 8) * 0x1p-24f;
}

/* Race uniform: odd multiples of 2^-24 in (0, 1), never 0 or 1, from the
 * low 23 bits of the Philox word (R6/R7). */
float oracle_u_race(uint32_t x)
{
    return (float)(2u * (x & 0x7FFFFFu) + 1u) * 0x1p-24f;
}

/* E(u) = -ln(u) rounded once to binary32 (R9).  The double log
 * is within a few ulp of exact, far inside the 74-ulp margin every u on the
 * race grid keeps from a binary32 rounding midpoint (pinned exhaustively in
 * tests/test_oracle_uniforms.py), so this is the correctly rounded value.   */
float oracle_E(float u)
{
    return (float)(-log((double)u));
}

void oracle_E_table(float* out /* [2^23] */)
{
    uint32_t m;
    for (m = 0; m < (1u << 23); ++m)
        out[m] = oracle_E((float)(2u * m + 1u) * 0x1p-24f);
}

/* ------------------------------------------------------------------------ */
/* Verify / accept: speculative sampling (Leviathan et al. 2023, Chen et al.
 * 2023; the paper's "we utilize rejection sampling to determine which tokens
 * are retained ... a bonus token that either rectifies an incorrect draft
 * prediction or extends the sequence", PAPER.md:18 [AD]; m+1 tokens with
 * minimum 1 and maximum k+1, PAPER.md:493-497 [BG]).
 *
 * For request i with k_i drafts x_0..x_{k-1}, target rows p_0..p_k and
 * draft rows q_0..q_{k-1} (q == NULL: one-hot drafts):
 *   1. for j = 0..k-1: accept x_j iff RN32(u_j * q_j[x_j]) < p_j[x_j]
 *      (i.e. with probability min(1, p/q)); m = first rejected j, else k.
 *   2. if m < k: w = max(0, p_m - q_m)   (residual, the correction)
 *      else     : w = max(0, p_k)        (the bonus token)
 *      if every w is 0: w = max(0, p_m)  (reading R5)
 *   3. t = argmax_v RN32(w_v / E(u_v)) over w_v > 0, lowest v on ties:
 *      the exponential race draws v with probability w_v / sum(w) (R7).
 *   4. emit x_0..x_{m-1}, t; num_accepted = m.
 * Injected uniforms (tests): inj_u_acc[R_q] replaces u_j, inj_E[R_p * V]
 * replaces E(u) of row r at column v.                                      */
/* ------------------------------------------------------------------------ */
static int32_t race_row(const float* pm, const float* qm, int32_t x_onehot, int32_t residual,
                        int32_t V, uint64_t seed, uint32_t step, uint32_t rid, int32_t m,
                        const float* inj_E_row)
{
    int32_t best = -1, v;
    float s_best = 0.0f;
    for (v = 0; v < V; ++v) {
        float w;
        if (residual) {
            float qv = qm ? qm[v] : (v == x_onehot ? 1.0f : 0.0f);
            float d = pm[v] - qv;
            w = (d > 0.0f) ? d : 0.0f;
        } else {
            w = (pm[v] > 0.0f) ? pm[v] : 0.0f;
        }
        if (w > 0.0f) {
            float E, s;
            if (inj_E_row) {
                E = inj_E_row[v];
            } else {
                uint32_t x = philox_word(seed, (uint32_t)v >> 2, 1u, (uint32_t)m, rid, step,
                                         (uint32_t)v & 3u);
                E = oracle_E(oracle_u_race(x));
            }
            s = w / E;
            if (best < 0 || s > s_best) { /* strict: lowest index wins ties */
                best = v;
                s_best = s;
            }
        }
    }
    return best;
}

int32_t oracle_verify(const float* p, const float* q, int64_t ld, int32_t V,
                      const int32_t* row_offsets, const int32_t* draft_tokens,
                      const uint32_t* request_ids, uint64_t seed, uint32_t step,
                      int32_t B, int32_t k_max,
                      const float* inj_u_acc, const float* inj_E,
                      int32_t* num_accepted, int32_t* out_tokens)
{
    int32_t status = 0, i, j;
    for (i = 0; i < B; ++i) {
        int32_t r0 = row_offsets[i], r1 = row_offsets[i + 1];
        int32_t k = r1 - r0 - 1;
        int32_t qbase = r0 - i; /* q rows and drafts of request i start here */
        int32_t m, t, bad = 0;
        uint32_t rid = request_ids[i];
        int32_t* out = out_tokens + (int64_t)i * (k_max + 1);
        for (j = 0; j <= k_max; ++j) out[j] = -1;
        num_accepted[i] = -1;
        if (k < 0 || k > k_max || qbase < 0) {
            status |= ORACLE_STATUS_BAD_K;
            continue;
        }
        for (j = 0; j < k; ++j) {
            int32_t x = draft_tokens[qbase + j];
            if (x < 0 || x >= V) bad = 1;
        }
        if (bad) {
            status |= ORACLE_STATUS_BAD_TOKEN;
            continue;
        }
        /* 1. acceptance test with first-rejection scan */
        m = k;
        for (j = 0; j < k; ++j) {
            int32_t x = draft_tokens[qbase + j];
            float u, qx, px, uq;
            if (inj_u_acc)
                u = inj_u_acc[qbase + j];
            else
                u = oracle_u_acc(philox_word(seed, 0u, 0u, (uint32_t)j, rid, step, 0u));
            qx = q ? q[(int64_t)(qbase + j) * ld + x] : 1.0f;
            px = p[(int64_t)(r0 + j) * ld + x];
            uq = u * qx;
            if (!(uq < px)) { /* strict; NaN rejects */
                m = j;
                break;
            }
        }
        /* 2-3. correction (residual) or bonus draw by exponential race */
        {
            const float* pm = p + (int64_t)(r0 + m) * ld;
            const float* qm = (m < k && q) ? q + (int64_t)(qbase + m) * ld : NULL;
            int32_t xm = (m < k) ? draft_tokens[qbase + m] : -1;
            const float* inj_row = inj_E ? inj_E + (int64_t)(r0 + m) * V : NULL;
            t = race_row(pm, qm, xm, m < k, V, seed, step, rid, m, inj_row);
            if (t < 0 && m < k) /* residual identically zero: fall back to p_m */
                t = race_row(pm, NULL, -1, 0, V, seed, step, rid, m, inj_row);
            if (t < 0) status |= ORACLE_STATUS_NO_WEIGHT;
        }
        /* 4. emit */
        for (j = 0; j < m; ++j) out[j] = draft_tokens[qbase + j];
        out[m] = t;
        num_accepted[i] = m;
    }
    return status;
}

/* ------------------------------------------------------------------------ */
/* Prompt lookup decoding (PAPER.md:57 [AD] "each request attempts to
 * retrieve a predetermined number of tokens ... proposal cost only depends on
 * the context search"; "proposed tokens are retrieved as
 * n-grams from the input prompt"; "uses the best matching
 * n-token string"; Fig. propose-verify-len: a request with no
 * match proposes nothing).  Reading R20: for n = n_max down to n_min, the
 * latest start s < L-n with ctx[s..s+n-1] == ctx[L-n..L-1]; propose
 * ctx[s+n .. min(s+n+K, L)-1]; no match for any n => length 0.            */
/* Greedy verification (temperature 0): the paper's dynamic-
 * workload and appendix runs use greedy decoding, under which
 * speculative decoding keeps a draft token iff it is the target's argmax, and the
 * correction / bonus token is the target's argmax at the first position that does not
 * match (or after the last draft).  Reading (R24): argmax over v < V of the
 * float values, NaN never selected, ties -> lowest index; a row with no non-NaN value has
 * no argmax (token -1, NO_WEIGHT).  Written out as the definition: one loop per row. */
static int32_t greedy_argmax(const float* row, int32_t V)
{
    int32_t v, best = -1;
    for (v = 0; v < V; ++v) {
        if (row[v] != row[v]) continue;            /* NaN */
        if (best < 0 || row[v] > row[best]) best = v;  /* strict: first maximum wins */
    }
    return best;
}

int32_t oracle_verify_greedy(const float* p, int64_t ld, int32_t V, const int32_t* row_offsets,
                             const int32_t* draft_tokens, int32_t B, int32_t k_max,
                             int32_t* num_accepted, int32_t* out_tokens)
{
    int32_t status = 0, i, j;
    for (i = 0; i < B; ++i) {
        int32_t r0 = row_offsets[i], r1 = row_offsets[i + 1];
        int32_t k = r1 - r0 - 1, qbase = r0 - i, m, t, bad = 0;
        int32_t* out = out_tokens + (int64_t)i * (k_max + 1);
        for (j = 0; j <= k_max; ++j) out[j] = -1;
        num_accepted[i] = -1;
        if (k < 0 || k > k_max || qbase < 0) {
            status |= ORACLE_STATUS_BAD_K;
            continue;
        }
        for (j = 0; j < k; ++j) {
            int32_t x = draft_tokens[qbase + j];
            if (x < 0 || x >= V) bad = 1;
        }
        if (bad) {
            status |= ORACLE_STATUS_BAD_TOKEN;
            continue;
        }
        m = k;  /* accept while the draft is the target's argmax */
        for (j = 0; j < k; ++j)
            if (draft_tokens[qbase + j] != greedy_argmax(p + (int64_t)(r0 + j) * ld, V)) {
                m = j;
                break;
            }
        t = greedy_argmax(p + (int64_t)(r0 + m) * ld, V);  /* correction (m < k) or bonus (m = k) */
        for (j = 0; j < m; ++j) out[j] = draft_tokens[qbase + j];
        out[m] = t;
        num_accepted[i] = m;
        if (t < 0) status |= ORACLE_STATUS_NO_WEIGHT;
    }
    return status;
}

/* Softmax from logits with temperature (reading R23: "p = softmax(z)
 * with fp32 exp, fp64 row sums"; the sampler of PAPER.md:493 receives the target / draft
 * distributions, which a serving stack holds as logits).  Per row, written out:
 *   inv_tau = RN32(1 / tau);  M = max_{v<V} z_v;
 *   e_v = expf(RN32(RN32(z_v - M) * inv_tau));  S = sum_v e_v in binary64 (ascending v);
 *   inv_S = RN32(1 / S);  p_v = RN32(e_v * inv_S).
 * Logits are finite or -inf, at least one finite per row.  The verify of R1-R9 then runs on
 * these p (and q) rows. */
void oracle_softmax_rows(const float* z, int64_t ld, int32_t V, int32_t rows, float temperature,
                         float* p_out)
{
    int32_t r, v;
    const float inv_tau = (float)(1.0 / (double)temperature);
    for (r = 0; r < rows; ++r) {
        const float* zr = z + (int64_t)r * ld;
        float* pr = p_out + (int64_t)r * ld;
        float M = zr[0], inv_S;
        double S = 0.0;
        for (v = 1; v < V; ++v)
            if (zr[v] > M) M = zr[v];
        for (v = 0; v < V; ++v) {
            float d = zr[v] - M;
            float a = d * inv_tau;
            S += (double)expf(a);
        }
        inv_S = (float)(1.0 / S);
        for (v = 0; v < V; ++v) {
            float d = zr[v] - M;
            float a = d * inv_tau;
            pr[v] = expf(a) * inv_S;
        }
        for (v = V; v < ld; ++v) pr[v] = 0.0f;
    }
}

/* Latency-model fit ("fits a linear regression model", Eq. forward-time
 * T = a N_context + gamma N_batched + delta; reading R25 = SPEC.md:44-52): ordinary least
 * squares on the columns (context, batched, 1); while a free coefficient is negative, clamp
 * every negative one to 0 and refit the remaining free ones.  R^2 = 1 - SS_res / SS_tot of the
 * final fit (1 when SS_tot = 0 and the fit is exact).  Returns 0, 1 (n < 3) or 2 (the full
 * design is rank-deficient).  Written out: normal equations, Gaussian elimination with
 * partial pivoting, in double. */
static int solve_normal(const double* X[3], const double* y, int32_t n, const int free_[3], double beta[3])
{
    double A[3][4];
    int idx[3], m = 0, i, j, c, r;
    for (i = 0; i < 3; ++i)
        if (free_[i]) idx[m++] = i;
    for (i = 0; i < m; ++i) {
        for (j = 0; j < m; ++j) {
            double s = 0.0;
            for (r = 0; r < n; ++r) s += X[idx[i]][r] * X[idx[j]][r];
            A[i][j] = s;
        }
        {
            double s = 0.0;
            for (r = 0; r < n; ++r) s += X[idx[i]][r] * y[r];
            A[i][m] = s;
        }
    }
    for (c = 0; c < m; ++c) {
        int piv = c;
        double scale = 0.0;
        for (r = 0; r < m; ++r)
            for (j = 0; j < m; ++j) scale = fabs(A[r][j]) > scale ? fabs(A[r][j]) : scale;
        for (r = c + 1; r < m; ++r)
            if (fabs(A[r][c]) > fabs(A[piv][c])) piv = r;
        if (!(fabs(A[piv][c]) > 1e-12 * scale)) return 2;
        if (piv != c)
            for (j = 0; j <= m; ++j) {
                double t = A[c][j];
                A[c][j] = A[piv][j];
                A[piv][j] = t;
            }
        for (r = c + 1; r < m; ++r) {
            double f = A[r][c] / A[c][c];
            for (j = c; j <= m; ++j) A[r][j] -= f * A[c][j];
        }
    }
    for (i = 0; i < 3; ++i) beta[i] = 0.0;
    for (c = m - 1; c >= 0; --c) {
        double s = A[c][m];
        for (j = c + 1; j < m; ++j) s -= A[c][j] * beta[idx[j]];
        beta[idx[c]] = s / A[c][c];
    }
    return 0;
}

int32_t oracle_fit_latency(const double* ctx_tokens, const double* batched_tokens, const double* ms, int32_t n,
                           double out[3], double* r2)
{
    double* ones;
    const double* X[3];
    int free_[3] = {1, 1, 1}, i, any_neg, st;
    double beta[3], mean = 0.0, ss_tot = 0.0, ss_res = 0.0;
    int32_t r;
    if (n < 3) return 1;
    ones = (double*)malloc(sizeof(double) * (size_t)n);
    for (r = 0; r < n; ++r) ones[r] = 1.0;
    X[0] = ctx_tokens;
    X[1] = batched_tokens;
    X[2] = ones;
    st = solve_normal(X, ms, n, free_, beta);
    if (st) {
        free(ones);
        return 2;
    }
    do {
        any_neg = 0;
        for (i = 0; i < 3; ++i)
            if (free_[i] && beta[i] < 0.0) {
                free_[i] = 0;
                any_neg = 1;
            }
        if (any_neg) {
            if (!free_[0] && !free_[1] && !free_[2]) {
                beta[0] = beta[1] = beta[2] = 0.0;
                break;
            }
            solve_normal(X, ms, n, free_, beta);
        }
    } while (any_neg);
    for (r = 0; r < n; ++r) mean += ms[r];
    mean /= (double)n;
    for (r = 0; r < n; ++r) {
        double pred = beta[0] * ctx_tokens[r] + beta[1] * batched_tokens[r] + beta[2];
        ss_res += (ms[r] - pred) * (ms[r] - pred);
        ss_tot += (ms[r] - mean) * (ms[r] - mean);
    }
    *r2 = ss_tot > 0.0 ? 1.0 - ss_res / ss_tot : (ss_res == 0.0 ? 1.0 : 0.0);
    for (i = 0; i < 3; ++i) out[i] = beta[i];
    free(ones);
    return 0;
}

/* Closed-loop harness (reading R26): the synthetic target model that
 * stands in for the LLM forward in a multi-step on-device loop, and the context append.
 * Not from the paper (which runs real models); a world in which every draft token is kept by
 * rejection sampling with probability exactly alpha_true:
 *   request i verifies k_i = k_req[i] drafts x_j = proposals[i][j] (j < k_i);
 *   row_offsets = exclusive scan of (k_i + 1); drafts packed at row_offsets[i] - i;
 *   row j < k_i:  p[x_j] = alpha_true, every other token (1 - alpha_true) / (V - 1) (V > 1);
 *   row k_i (bonus): uniform 1 / V.
 * With one-hot drafts (q = NULL) the acceptance test is u < p[x_j] = alpha_true. */
void oracle_sim_target(const int32_t* proposals, int32_t K, const int32_t* k_req, int32_t B, float alpha_true,
                       int32_t V, int64_t ld, float* p_out, int32_t* row_offsets, int32_t* drafts)
{
    int32_t i, j, v, r = 0;
    const float rest = V > 1 ? (float)((1.0 - (double)alpha_true) / (double)(V - 1)) : 0.0f;
    const float unif = (float)(1.0 / (double)V);
    for (i = 0; i < B; ++i) {
        int32_t k = k_req[i];
        row_offsets[i] = r;
        for (j = 0; j <= k; ++j, ++r) {
            float* row = p_out + (int64_t)r * ld;
            if (j < k) {
                int32_t x = proposals[(int64_t)i * K + j];
                drafts[r - i] = x;
                for (v = 0; v < V; ++v) row[v] = rest;
                row[x] = alpha_true;
            } else {
                for (v = 0; v < V; ++v) row[v] = unif;
            }
        }
    }
    row_offsets[B] = r;
}

/* Context window of L tokens per request (request i at [i L, (i+1) L)): the m_i + 1 emitted
 * tokens are appended and as many of the oldest dropped; ctx_len[i] (the context length the
 * latency model sees) grows by m_i + 1.  A request with m_i < 0 (flagged) is unchanged. */
void oracle_context_append(const int32_t* ctx_in, int32_t L, int32_t B, const int32_t* out_tokens,
                           const int32_t* num_accepted, int32_t k_max, int32_t* ctx_out, int32_t* ctx_len)
{
    int32_t i, t;
    for (i = 0; i < B; ++i) {
        int32_t e = num_accepted[i] >= 0 ? num_accepted[i] + 1 : 0;
        const int32_t* in = ctx_in + (int64_t)i * L;
        int32_t* out = ctx_out + (int64_t)i * L;
        if (e > L) e = L;
        for (t = 0; t < L - e; ++t) out[t] = in[t + e];
        for (t = 0; t < e; ++t) out[L - e + t] = out_tokens[(int64_t)i * (k_max + 1) + (num_accepted[i] + 1 - e) + t];
        ctx_len[i] += num_accepted[i] >= 0 ? num_accepted[i] + 1 : 0;
    }
}

/* ------------------------------------------------------------------------ */
void oracle_lookup(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                   int32_t n_min, int32_t n_max, int32_t K,
                   int32_t* proposals, int32_t* proposal_len)
{
    int32_t i;
    for (i = 0; i < B; ++i) {
        const int32_t* c = ctx + ctx_offsets[i];
        int32_t L = ctx_offsets[i + 1] - ctx_offsets[i];
        int32_t* prop = proposals + (int64_t)i * K;
        int32_t n, s, t, len = 0, found = 0;
        for (t = 0; t < K; ++t) prop[t] = -1;
        for (n = n_max; n >= n_min && !found; --n) {
            if (L < n + 1) continue;
            for (s = L - n - 1; s >= 0; --s) {
                int32_t match = 1;
                for (t = 0; t < n; ++t) {
                    if (c[s + t] != c[L - n + t]) { match = 0; break; }
                }
                if (match) {
                    int32_t end = s + n + K;
                    if (end > L) end = L;
                    for (t = s + n; t < end; ++t) prop[len++] = c[t];
                    found = 1;
                    break;
                }
            }
        }
        proposal_len[i] = len;
    }
}

/* ------------------------------------------------------------------------ */
/* Goodput adaptor.                                                          */
/* ------------------------------------------------------------------------ */

/* Eq. gen_len (PAPER.md:133-139 [AD]): l(a, k) = (1 - a^{k+1}) / (1 - a) =
 * sum_{j=0..k} a^j, evaluated by Horner as 1 + a(1 + a(1 + ...)) with an
 * explicit fma per step (reading R11: the limit k+1 at a = 1, no division). */
double oracle_expected_len(double alpha, int32_t k)
{
    double acc = 1.0;
    int32_t j;
    for (j = 0; j < k; ++j) acc = fma(alpha, acc, 1.0);
    return acc;
}

/* Eq. forward-time (PAPER.md:106-113 [AD]):
 * T_fwd = a * N_context + gamma * N_batched + delta, evaluated as
 * fma(gamma, N_batched, fma(a, N_context, delta)).                         */
double oracle_forward_time(const double model[3], double n_context, double n_batched)
{
    return fma(model[1], n_batched, fma(model[0], n_context, model[2]));
}

/* ArgMaxGoodput, Listing 2 (PAPER.md:256-270 [AD]) with Eq. goodput
 * (PAPER.md:38-42), Eq. batch-latency, T_draft = s*T_fwd
 * and the batch sum of Eq. gen_len.
 * Readings: R12 (k = 0 searched, strict >), R13 (k_i = min(k, cap_i)),
 * R14 (OOM = sum(k_i+1) > kv_free), R15/R16 (draft / PLD cost), fixed-point
 * token sums.  Returns k*.                            */
int32_t oracle_choose_k(const double* alpha, int32_t alpha_per_request,
                        const int32_t* ctx_len, const int32_t* cap, int32_t B, int32_t k_max,
                        int32_t policy, const double target[3], const double draft[3],
                        double pld_cost_ms, int64_t kv_free_slots, double* goodput_out)
{
    double max_goodput = -1.0;
    int32_t best_k = 0, k, i;
    int64_t n_ctx = 0, n_ctx_spec = 0, b_spec = 0;
    for (i = 0; i < B; ++i) {
        n_ctx += ctx_len[i];
        if (cap[i] > 0) {
            n_ctx_spec += ctx_len[i];
            b_spec += 1;
        }
    }
    for (k = 0; k <= k_max; ++k) {
        int64_t l_fixed = 0, n_batched = 0;
        double t_target, t_draft, goodput;
        for (i = 0; i < B; ++i) {
            int32_t ki = k < cap[i] ? k : cap[i];
            double a = alpha_per_request ? alpha[i] : alpha[0];
            if (ki < 0) ki = 0;
            l_fixed += llrint(ldexp(oracle_expected_len(a, ki), 32));
            n_batched += (int64_t)ki + 1;
        }
        if (k > 0 && kv_free_slots >= 0 && n_batched > kv_free_slots) {
            if (goodput_out) goodput_out[k] = -1.0;
            continue; /* Listing 2 line 5: OOM(proposed_cnt) -> continue */
        }
        t_target = oracle_forward_time(target, (double)n_ctx, (double)n_batched);
        if (policy == ORACLE_POLICY_PLD)
            t_draft = pld_cost_ms;
        else
            t_draft = (k > 0) ? (double)k * oracle_forward_time(draft, (double)n_ctx_spec, (double)b_spec)
                              : 0.0;
        goodput = ldexp((double)l_fixed, -32) / (t_target + t_draft);
        if (goodput_out) goodput_out[k] = goodput;
        if (goodput > max_goodput) {
            max_goodput = goodput;
            best_k = k;
        }
    }
    return best_k;
}

/* UpdateGlobalAcceptance (Listing 1 line 19) with the moving
 * average of PAPER.md:131-132: alpha' = d*alpha + (1-d)*r evaluated as
 * fma(d, alpha - r, r) (reading R17), r = sum(m) / sum(tested) (R18;
 * estimator PROPOSED uses sum(k)).  A step with nothing tested leaves alpha.
 * per_request != 0: alpha[i] updated from request i alone (R19).           */
void oracle_update(double* alpha, int32_t per_request, const int32_t* num_accepted,
                   const int32_t* row_offsets, int32_t B, double decay, int32_t estimator)
{
    int64_t sum_m = 0, sum_t = 0;
    int32_t i;
    for (i = 0; i < B; ++i) {
        int32_t k = row_offsets[i + 1] - row_offsets[i] - 1;
        int32_t m = num_accepted[i];
        int64_t t;
        if (m < 0) continue; /* invalid request (status set by verify) */
        t = (estimator == ORACLE_EST_PROPOSED) ? k : (m + (m < k ? 1 : 0));
        if (per_request) {
            if (t > 0) {
                double r = (double)m / (double)t;
                alpha[i] = fma(decay, alpha[i] - r, r);
            }
        } else {
            sum_m += m;
            sum_t += t;
        }
    }
    if (!per_request && sum_t > 0) {
        double r = (double)sum_m / (double)sum_t;
        alpha[0] = fma(decay, alpha[0] - r, r);
    }
}
