// verify.cu -- rejection-sampling verify/accept on sm_100a.
// PAPER.md:18 [AD], 493-497 [BG]; readings R1-R9 in DESIGN.md section 3.
//
// One tsv_verify_accept call = three kernels chained with programmatic dependent launch
// (PDL, griddepcontrol), so each kernel's launch and prologue overlap its predecessor:
//
//  1. verify_scan_kernel: one warp per request.  Acceptance test with first-rejection
//     scan (lane j < k_i gathers p_j[x_j], q_j[x_j], draws u_acc, one ballot) -> m_i.
//     Writes a 32-byte ReqMeta per request and m_i; bad requests are emitted (-1) here.
//  2. verify_race_kernel: warp-independent.  Work item = (request, column chunk; the
//     default chunk gives about one item per resident warp) of the selected row [lazy] or
//     (request, position, chunk) of every row [vocab-shard partial], request-minor over
//     all warps of the grid.  Each warp streams its chunk of p -- and of q on a rejection --
//     two 128-bit loads per lane per step, one specialised Philox4x32-10 call per float4,
//     the provably conservative prune test that skips the exact
//     double-log + IEEE-division score of elements that cannot reach the best score seen,
//     deferred exact evaluation of survivors, and a packed (score, ~index) u64 key per
//     row combined with red.max.  No shared memory, no barriers in the race itself; with
//     tsv_verify_accept_update the grid's item-less last warp (else one extra CTA) runs the
//     alpha update beside the race (the accepted counts are final after the scan).
//  3. verify_emit_kernel: one warp per request (or p row in shard mode) reads the row key,
//     falls back to the p_m race when the residual was identically zero (R5), and emits
//     the correction / bonus token (or the shard tuple).
// Also here: the lazy two-round vocab sharding kernels (flags / meta / keys / emit), the
// greedy verify (dense row argmax + first-mismatch emit), the fused softmax-from-logits
// verify (online-softmax partials + logits scan; the race and emit take a LOGITS flag),
// the standalone softmax rows, and the injected-word race diagnostic.
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "goodput.cuh"
#include "p2p.cuh"

namespace tsv {

struct ReqMeta {           // 32 bytes, written by the scan kernel
    int32_t r0, k, qbase, m;
    int32_t xm, ok;        // ok: 1 valid, 0 bad k, 2 bad draft token
    uint32_t rid, pad;     // pad: the call's epoch in the p2p modes (0 otherwise)
};

struct RaceParams {
    const float* p;
    const float* q;
    const int32_t* row_offsets;
    const int32_t* drafts;
    const uint32_t* rids;
    int32_t* num_accepted;
    int32_t* out_tokens;
    int32_t* devstatus;
    long long* step_counts;    // nullable: (sum m_i, sum tested_i) over valid requests (tsv_verify_args)
    ReqMeta* meta;             // [B]
    uint32_t* rowT;            // [n_key_rows] shared race threshold per raced row (float bits)
    unsigned long long* rowkey;  // [n_key_rows] max race key per raced row (0: nothing evaluated)
    tsv_shard_tuple* tuples;   // shard mode
    const float4* lstats;      // logits mode: per request (M_p, 1/S_p, M_q, 1/S_q) of row m
    float inv_tau;             // logits mode: RN32(1 / temperature)
    int64_t ld;
    uint32_t k0, k1, step;
    int32_t B, k_max, vocab, vocab_offset, vocab_global, chunk, n_chunks, rows_p;
    uint32_t ks0[10], ks1[10];  // Philox key schedule k + r W (constant bank)
    int32_t meta_ready;         // TSV_VERIFY_META_READY: the scan reads row_offsets/drafts/rids before its wait
    int32_t early_trigger;      // TSV_VERIFY_EARLY_TRIGGER: the emit kernel triggers its dependents before its wait
    uint32_t* alpha_ready;      // nullable (tsv_verify_accept_update_ex): reset to 0 by the scan, set by the update
    int32_t race_update;        // lazy race: the alpha update (ua) beside the race (1: extra CTA, 2: last warp)
    UpdateArgs ua;
    int32_t push;               // TSV_VERIFY_P2P_FUSED: each race item pushes its chunk key to every rank (pv)
    P2PView pv;
};

enum Mode { kLazy = 0, kShard = 1 };

// Logits mode (reading R23): p = RN32(expf(RN32(RN32(z - M) * inv_tau)) * inv_S), CUDA's
// accurate expf (<= 2 ulp; the oracle's glibc expf is correctly rounded).
__device__ __forceinline__ float to_prob(float z, float M, float inv_S, float inv_tau) {
    return __fmul_rn(expf(__fmul_rn(__fsub_rn(z, M), inv_tau)), inv_S);
}
__device__ __forceinline__ float4 to_prob4(const float4& z, float M, float inv_S, float inv_tau) {
    return make_float4(to_prob(z.x, M, inv_S, inv_tau), to_prob(z.y, M, inv_S, inv_tau),
                       to_prob(z.z, M, inv_S, inv_tau), to_prob(z.w, M, inv_S, inv_tau));
}

constexpr int kMaxChunk = 16384;
constexpr float kPruneC = 0x1.fffffap-1f;        // 1 - 3*2^-24 <= (1-2^-23)(1-2^-24)
constexpr float kLbC = 0x1.ffffe0p-1f;           // 1 - 2^-20
constexpr float kMinNormal = 0x1p-126f;


// Lower bound on the exact score RN32(w / E(u)) of an element:
// E <= (-ln u)(1+2^-24) <= ((1-u)/u)(1+2^-24), and rcp.approx is within 2^-22.
__device__ __forceinline__ float race_lower_bound(float w, float omu) {
    const float u = __fsub_rn(1.0f, omu);  // exact
    return __fmul_rd(__fmul_rd(w, u), __fmul_rd(rcp_approx(omu), kLbC));
}

#ifndef TSV_SCAN_PREFETCH
#define TSV_SCAN_PREFETCH 1
#endif
#ifndef TSV_UPDATE_WARP
#define TSV_UPDATE_WARP 1
#endif
#ifndef TSV_RACE_FTZ
#define TSV_RACE_FTZ 1
#endif
__device__ __forceinline__ float prune_scale(float T) {
#if TSV_RACE_FTZ
    // one flush-to-zero multiply: a subnormal T, or a product below the normal range, gives Tc = 0
    // (nothing with w > 0 is skipped), as conservative as the explicit test it replaces
    float r;
    asm("mul.rm.ftz.f32 %0, %1, %2;" : "=f"(r) : "f"(T), "f"(kPruneC));
    return r;
#else
    return T >= kMinNormal ? __fmul_rd(T, kPruneC) : 0.0f;
#endif
}

// Packed fp32 pairs (sm_100 FADD2 / FFMA2: two IEEE binary32 operations per instruction, each
// rounded exactly as its scalar form).
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 f2_unpack(uint64_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {  // RN(a - b) per lane
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ void f2_sub_if(uint64_t& a, uint64_t b, bool on) {  // a = RN(a - b) per lane if on
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q sub.rn.f32x2 %0, %0, %1;\n\t}"
        : "+l"(a)
        : "l"(b), "r"(static_cast<uint32_t>(on)));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {  // RN(a b + c) per lane
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

struct Race;
#ifndef TSV_COUNT_EXACT
#define TSV_COUNT_EXACT 0
#endif
#if TSV_COUNT_EXACT  // diagnostic builds only: exact evaluations / candidates / quads raced
__device__ unsigned long long g_exact_count[4];
#endif

// Per-thread race state.  T is warp-uniform: a lower bound on (or an exact value of) a
// score achieved by an element of this row.  Prune test: skipping element
// (w, u) is safe iff w <= Tc (1 - u) with Tc = RD(T (1 - 3 2^-24)).  With F = 1 - u + K,
// K = 1 - 2^-24 (race_F, exact), t = RN(Tc F - w) (one FFMA) and Th = RU(Tc (1 + 2^-23)),
// t >= Th implies Tc F - w >= Th - |t| 2^-24 >= Tc K, i.e. w <= Tc (1 - u): skip.  So an
// element is a candidate iff t < Th (3 instructions: LOP3, FFMA, FSETP); w <= 0 and NaN
// never pass the exact step (checked on the rare candidate path).
struct Race {
    float T, Tc, Th, Tloc;
    uint64_t best;
    // the parked candidate: pend_w > 0 iff one is parked (only w > 0 is ever parked); its 1 - u
    // determines E(u) exactly (race_E_omu), so the Philox word itself is not kept
    float pend_w, pend_omu;
    uint32_t pend_v;

    __device__ __forceinline__ void init() {
        T = Tc = Th = Tloc = 0.0f;
        best = 0;
        pend_w = 0.0f;
        pend_omu = 1.0f;
        pend_v = 0;
    }

    __device__ __forceinline__ void set_T(float t) {
        T = t;
        Tc = prune_scale(T);
        Th = __fmul_ru(Tc, 0x1.000002p+0f);
    }

    __device__ __forceinline__ void eval_exact(float w, float omu, uint32_t vg) {
#if TSV_COUNT_EXACT
        atomicAdd(&g_exact_count[0], 1ull);
#endif
        const uint64_t key = pack_key(__fdiv_rn(w, race_E_omu(omu)), vg);  // = exact_race_key(w, x, vg)
        best = key > best ? key : best;
        Tloc = fmaxf(Tloc, __uint_as_float(static_cast<uint32_t>(best >> 32)));
    }

    // Seed T from lower bounds of one float4 (first step of an item; warp-uniform call).
    __device__ __forceinline__ void warm(const float (&w)[4], const uint4& r) {
        const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
        float lb = 0.0f;
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (w[e] > 0.0f) lb = fmaxf(lb, race_lower_bound(w[e], one_minus_u_race(rw[e])));
        Tloc = fmaxf(Tloc, lb);
        sync_T();
    }

    // One float4 of weights w with Philox words r, global index v0.
    template <bool PRUNE>
    __device__ __forceinline__ void quad(const float (&w)[4], const uint4& r, uint32_t v0) {
        const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
        if constexpr (!PRUNE) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (w[e] > 0.0f) eval_exact(w[e], one_minus_u_race(rw[e]), v0 + e);
        } else {
            bool cand[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) cand[e] = __fmaf_rn(Tc, race_F(rw[e]), -w[e]) < Th;
#if TSV_COUNT_EXACT
            atomicAdd(&g_exact_count[2], 1ull);
            atomicAdd(&g_exact_count[1], static_cast<unsigned long long>(cand[0] + cand[1] + cand[2] + cand[3]));
#endif
            if (cand[0] | cand[1] | cand[2] | cand[3]) {
#if TSV_COUNT_EXACT
                if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicAdd(&g_exact_count[3], 32ull);  // warp entries
#endif
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (cand[e] && w[e] > 0.0f) {
                        const float omu = one_minus_u_race(rw[e]);
                        Tloc = fmaxf(Tloc, race_lower_bound(w[e], omu));
                        if (pend_w > __fmul_rd(Tc, pend_omu)) eval_exact(pend_w, pend_omu, pend_v);
                        pend_w = w[e];
                        pend_omu = omu;
                        pend_v = v0 + e;
                    }
                }
            }
        }
    }

    // The same race step with the prune values precomputed two at a time (TSV_RACE_F32X2):
    // s[e] = RN(w_e - Tc F_e) = -RN(Tc F_e - w_e) exactly (round-to-nearest is symmetric), so
    // "t < Th" is "s > -Th".
    // cu: the float4's Philox quad counter, vbase: the vocab offset; its global index is 4 cu + (vbase & 3),
    // formed on the candidate path only.
    __device__ __forceinline__ void quad_s(const float (&w)[4], const float (&sv)[4], const uint4& r, uint32_t cu,
                                           int32_t vbase) {
        const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
        const float nTh = -Th;
        if (fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3])) > nTh) {
#if TSV_COUNT_EXACT
            if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicAdd(&g_exact_count[3], 32ull);  // warp entries
#endif
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (sv[e] > nTh && w[e] > 0.0f) {
                    const float omu = one_minus_u_race(rw[e]);
                    Tloc = fmaxf(Tloc, race_lower_bound(w[e], omu));
                    if (pend_w > __fmul_rd(Tc, pend_omu)) eval_exact(pend_w, pend_omu, pend_v);
                    pend_w = w[e];
                    pend_omu = omu;
                    pend_v = 4u * cu + (static_cast<uint32_t>(vbase) & 3u) + e;
                }
            }
        }
#if TSV_COUNT_EXACT
        atomicAdd(&g_exact_count[2], 1ull);
        atomicAdd(&g_exact_count[1], static_cast<unsigned long long>((sv[0] > nTh) + (sv[1] > nTh) + (sv[2] > nTh) +
                                                                     (sv[3] > nTh)));
#endif
    }

    __device__ __forceinline__ void sync_T() {  // warp-wide max (REDUX on the float bits)
        set_T(__uint_as_float(__reduce_max_sync(0xFFFFFFFFu, __float_as_uint(Tloc))));
    }

    // Flush the parked candidate against a (possibly shared) final threshold.
    template <bool PRUNE>
    __device__ __forceinline__ void finish(float T_final) {
        if constexpr (PRUNE) {
            const float tc = prune_scale(T_final);
            if (pend_w > __fmul_rd(tc, pend_omu)) eval_exact(pend_w, pend_omu, pend_v);
            pend_w = 0.0f;
        }
    }
};

// Weights of one float4: residual p - q (dense q, or one-hot at local column xm) or bonus
// p; columns >= col_end are 0.  No max(0, .) clamp: the prune comparison rejects w <= 0
// and NaN (t < Th fails) and the candidate path re-checks w > 0, so max(0, p - q) of R1 is
// realised exactly.
template <bool DENSE_Q>
__device__ __forceinline__ void quad_weights(float (&w)[4], const float4& a, const float4& b, bool residual,
                                             int32_t col, int32_t col_end, int32_t xm) {
    const float pv[4] = {a.x, a.y, a.z, a.w};
    const float qv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) w[e] = pv[e];
    if (residual) {
        if (DENSE_Q) {
#pragma unroll
            for (int e = 0; e < 4; ++e) w[e] = __fsub_rn(pv[e], qv[e]);
        } else if ((col >> 2) == (xm >> 2)) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (col + e == xm) w[e] = __fsub_rn(pv[e], 1.0f);
        }
    }
    if (col + 4 > col_end) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (col + e >= col_end) w[e] = 0.0f;
    }
}

// Weights of one float4 in the streaming loop: p (w, already loaded), minus q (dense, when use_q) or
// minus the one-hot draft at local column xm (one-hot q on a rejection); col: the float4's local column.
template <bool DENSE_Q>
__device__ __forceinline__ void race_weights(float (&w)[4], const float4& b, bool use_q, bool residual, int32_t col,
                                             int32_t xm) {
    if (DENSE_Q) {
        if (use_q) {
            w[0] = __fsub_rn(w[0], b.x);
            w[1] = __fsub_rn(w[1], b.y);
            w[2] = __fsub_rn(w[2], b.z);
            w[3] = __fsub_rn(w[3], b.w);
        }
    } else if (residual && (col >> 2) == (xm >> 2)) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (col + e == xm) w[e] = __fsub_rn(w[e], 1.0f);
    }
}

// Request i's rows lie inside the allocations (tsv.h: device-side data errors): k_i in
// [0, k_max], its p rows r0 .. r1-1 below rows_lim, and its drafts / q rows qbase .. qbase+k-1
// (qbase = r0 - i) below rows_lim - B.  rows_lim is the host-known rows_p, or for the dense
// passes min(row_offsets[B], rows_p) -- the rows they actually covered.  int64: no overflow.
__device__ __forceinline__ bool request_rows_ok(int32_t r0, int32_t r1, int32_t i, int32_t k_max, int32_t rows_lim,
                                                int32_t B) {
    const int64_t k = static_cast<int64_t>(r1) - r0 - 1, qbase = static_cast<int64_t>(r0) - i;
    return k >= 0 && k <= k_max && qbase >= 0 && r1 <= rows_lim && qbase + k <= static_cast<int64_t>(rows_lim) - B;
}

// step_counts (tsv.h): (sum m_i, sum tested_i), tested_i = m_i + [m_i < k_i], over the valid
// requests of the call.  Zeroed by the call's first kernel (after its grid-dependency wait, so
// the previous call's adds are complete); the final kernel adds one shared-memory sum per CTA.
// Called by every thread of the CTA; `mine`: this thread carries request (m, k) (warp lane 0).
__device__ __forceinline__ void zero_step_counts(long long* sc) {
    if (sc && blockIdx.x == 0 && threadIdx.x == 0) {
        sc[0] = 0;
        sc[1] = 0;
    }
}
__device__ __forceinline__ void add_step_counts(long long* sc, bool mine, int32_t m, int32_t k) {
    __shared__ unsigned long long s_c[2];
    if (threadIdx.x == 0) s_c[0] = s_c[1] = 0ull;
    __syncthreads();
    if (mine && m >= 0) {
        atomicAdd(&s_c[0], static_cast<unsigned long long>(m));
        atomicAdd(&s_c[1], static_cast<unsigned long long>(m + (m < k ? 1 : 0)));
    }
    __syncthreads();
    if (threadIdx.x == 0 && (s_c[0] | s_c[1])) {
        atomicAdd(reinterpret_cast<unsigned long long*>(sc), s_c[0]);
        atomicAdd(reinterpret_cast<unsigned long long*>(sc) + 1, s_c[1]);
    }
}

// Rows covered by a dense pass over the batch: row_offsets[B] clamped to [0, rows_p].
__device__ __forceinline__ int32_t dense_rows(const int32_t* row_offsets, int32_t B, int32_t rows_p) {
    const int32_t r = row_offsets[B];
    return r < 0 ? 0 : (r > rows_p ? rows_p : r);
}

// Emit (R1-R4 step 4): lanes j <= k_max of one warp.
__device__ __forceinline__ void emit(const RaceParams& P, int32_t i, int32_t qbase, int32_t m, int32_t t) {
    const int lane = threadIdx.x & 31;
    int32_t* out = P.out_tokens + static_cast<int64_t>(i) * (P.k_max + 1);
    if (lane <= P.k_max) {
        int32_t v = -1;
        if (m >= 0) {
            if (lane < m) v = P.drafts[qbase + lane];
            else if (lane == m) v = t;
        }
        out[lane] = v;
    }
    if (lane == 0) P.num_accepted[i] = m;
}

// The scan's share of the emit (lazy modes): lanes j < m write the accepted drafts x_j
// (already in the lane's register), lanes m < j <= k_max the -1 padding.  Slot m (the
// correction / bonus token t) is left to the emit kernel, which then needs one load round
// trip (meta + row key) and one store.
__device__ __forceinline__ void emit_prefix(const RaceParams& P, int32_t i, int32_t m, int32_t x) {
    const int lane = threadIdx.x & 31;
    if (lane <= P.k_max && lane != m)
        P.out_tokens[static_cast<int64_t>(i) * (P.k_max + 1) + lane] = lane < m ? x : -1;
}

// ------------------------------------------------------------------ 1. acceptance scan
// One warp per request (R1-R4).  Lane j < k tests draft j if this shard owns x_j (the
// lazy mode's shard is the whole vocabulary).  Lazy: invalid requests are emitted here.
// Shard: writes the accept / owner flags of every p row of the request into its tuple.
template <int MODE>
__global__ void __launch_bounds__(256) verify_scan_kernel(const RaceParams P) {
    TSV_STEP_SPAN(2);
    // TSV_VERIFY_META_READY: row_offsets / draft_tokens / request_ids were not written by the
    // preceding kernel, so they are read while it drains; p and q only after the wait.
    if (!P.meta_ready) {
        pdl_wait();               // inputs of this step are complete
        TSV_STEP_WAITED();
        pdl_launch_dependents();  // let the race kernel launch and set up while we scan
    }
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const int lane = threadIdx.x & 31;
    const int32_t r0 = P.row_offsets[i];
    const int32_t r1 = P.row_offsets[i + 1];
    const int32_t k = r1 - r0 - 1;
    const int32_t qbase = r0 - i;
    int32_t ok = request_rows_ok(r0, r1, i, P.k_max, P.rows_p, P.B) ? 1 : 0;
    const uint32_t rid = P.rids[i];
    int32_t x = -1;
    bool bad = false, acc = false, own = false;
    if (ok && lane < k) x = P.drafts[qbase + lane];
    // everything that does not read p or q: with META_READY before the wait (the acceptance uniform too)
    const int32_t xl = x - P.vocab_offset;
    if (ok && lane < k) {
        bad = x < 0 || x >= P.vocab_global;
        own = !bad && xl >= 0 && xl < P.vocab;
    }
    float u = 0.0f;
    if (own) u = u_acc_from_word(philox4x32_10(0u, (kPurposeAccept << 16) | static_cast<uint32_t>(lane), rid, P.step,
                                               P.k0, P.k1).x);
    if (P.meta_ready) {
#if TSV_SCAN_PREFETCH
        // the words gathered below, into L2 while the previous kernel drains: a prefetch returns no data, and
        // every write reaches L2 (the coherence point), so what is read after the wait is what was written
        if (own) {
            prefetch_l2(P.p + static_cast<int64_t>(r0 + lane) * P.ld + xl);
            if (P.q) prefetch_l2(P.q + static_cast<int64_t>(qbase + lane) * P.ld + xl);
        }
#endif
        pdl_wait();
        TSV_STEP_WAITED();
        pdl_launch_dependents();
    }
    zero_step_counts(P.step_counts);
    if (P.alpha_ready && blockIdx.x == 0 && threadIdx.x == 0) *P.alpha_ready = 0u;  // alpha of this call: pending
    if (own) {
        const float qx = P.q ? P.q[static_cast<int64_t>(qbase + lane) * P.ld + xl] : 1.0f;
        const float px = P.p[static_cast<int64_t>(r0 + lane) * P.ld + xl];
        acc = __fmul_rn(u, qx) < px;  // strict; NaN rejects
    }
    const uint32_t badm = __ballot_sync(0xFFFFFFFFu, bad);
    const uint32_t accm = __ballot_sync(0xFFFFFFFFu, acc);
    const uint32_t ownm = __ballot_sync(0xFFFFFFFFu, own);
    if (badm) ok = 2;
    const uint32_t kmask = (ok == 1 && k > 0) ? ((1u << k) - 1u) : 0u;
    const uint32_t rej = ~accm & kmask;
    const int32_t m = rej ? (__ffs(rej) - 1) : (ok == 1 ? k : -1);
    const int32_t xm = __shfl_sync(0xFFFFFFFFu, x, (m >= 0 ? m : 0) & 31);
    if (MODE == kLazy) {
        if (lane == 0) {
            P.rowT[i] = 0u;
            P.rowkey[i] = 0ull;
        }
    } else if (ok == 1 && lane <= k) {
        P.rowT[r0 + lane] = 0u;
        P.rowkey[r0 + lane] = 0ull;
    }
    if (lane == 0) {
        ReqMeta rm;
        rm.r0 = r0;
        rm.k = k;
        rm.qbase = qbase;
        rm.m = m;
        rm.xm = (m >= 0 && m < k) ? xm : -1;
        rm.ok = ok;
        rm.rid = rid;
        rm.pad = 0;
        P.meta[i] = rm;
    }
    if (MODE == kLazy) {
        if (lane == 0) P.num_accepted[i] = m;  // final here (-1: bad request); the update may read it
        if (ok == 1) emit_prefix(P, i, m, x);
        else {
            emit(P, i, 0, -1, -1);
            if (lane == 0) report(P.devstatus, ok == 2 ? TSV_DEVSTATUS_BAD_TOKEN : TSV_DEVSTATUS_BAD_K);
        }
    } else if (ok == 1 && lane <= k) {  // rows j <= k of this request: flags (bit0 accept, bit1 owner)
        const uint32_t flag = lane < k ? (((accm >> lane) & 1u) | (((ownm >> lane) & 1u) << 1)) : 0u;
        P.tuples[r0 + lane].flag = flag;
        P.tuples[r0 + lane].pad = 0;
    }
}

// UpdateGlobalAcceptance (Listing 1 line 19) over one CTA of any size (all threads call):
// exact int64 sums of m and tested, then the EWMA -- the arithmetic of update_block.
__device__ __forceinline__ void update_cta(const UpdateArgs& A) {
    __shared__ long long red2[32][2];
    long long sm = 0, stt = 0;
    for (int32_t i = threadIdx.x; i < A.B; i += blockDim.x) {
        const int32_t k = A.row_offsets[i + 1] - A.row_offsets[i] - 1;
        const int32_t m = __ldcg(A.num_accepted + i);
        if (m < 0) continue;
        const long long t = A.estimator == TSV_EST_PROPOSED ? k : (m + (m < k ? 1 : 0));
        if (A.per_request) {
            if (t > 0) {
                const double r = __ddiv_rn(static_cast<double>(m), static_cast<double>(t));
                A.alpha[i] = __fma_rn(A.decay, __dsub_rn(A.alpha[i], r), r);
            }
        } else {
            sm += m;
            stt += t;
        }
    }
    if (A.per_request) {
        if (A.alpha_ready) {  // every thread wrote its alpha_i: publish them together
            __syncthreads();
            if (threadIdx.x == 0) signal_alpha_ready(A.alpha_ready);
        }
        return;
    }
    sm = warp_sum_i64(sm);
    stt = warp_sum_i64(stt);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        red2[warp][0] = sm;
        red2[warp][1] = stt;
    }
    __syncthreads();
    __shared__ long long s_ab[2];
    if (threadIdx.x == 0) {
        long long a = 0, b = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            a += red2[w][0];
            b += red2[w][1];
        }
        if (!A.use_p2p) {
            ewma_apply(A.alpha, a, b, A.decay);
            signal_alpha_ready(A.alpha_ready);
        }
        s_ab[0] = a;
        s_ab[1] = b;
    }
    if (A.use_p2p) {  // request-sharded global alpha: sum the pair over the ranks (p2p.cuh), same EWMA everywhere
        __syncthreads();
        p2p_allreduce_block(s_ab, 2, A.p2p, A.devstatus);
        if (threadIdx.x == 0) {
            ewma_apply(A.alpha, s_ab[0], s_ab[1], A.decay);
            signal_alpha_ready(A.alpha_ready);
        }
    }
}

// The same update run by ONE warp (the race grid's last warp when it has no work item, so the update
// needs no extra CTA whatever the race's CTA shape): identical sums, EWMA and alpha_ready signal.
__device__ __forceinline__ void update_warp(const UpdateArgs& A) {
    const int lane = threadIdx.x & 31;
    long long sm = 0, stt = 0;
    for (int32_t i = lane; i < A.B; i += 32) {
        const int32_t k = A.row_offsets[i + 1] - A.row_offsets[i] - 1;
        const int32_t m = __ldcg(A.num_accepted + i);
        if (m < 0) continue;
        const long long t = A.estimator == TSV_EST_PROPOSED ? k : (m + (m < k ? 1 : 0));
        if (A.per_request) {
            if (t > 0) {
                const double r = __ddiv_rn(static_cast<double>(m), static_cast<double>(t));
                A.alpha[i] = __fma_rn(A.decay, __dsub_rn(A.alpha[i], r), r);
            }
        } else {
            sm += m;
            stt += t;
        }
    }
    if (A.per_request) {
        if (A.alpha_ready) {  // every lane wrote its alpha_i: publish them together
            __syncwarp();
            if (lane == 0) signal_alpha_ready(A.alpha_ready);
        }
        return;
    }
    sm = warp_sum_i64(sm);
    stt = warp_sum_i64(stt);
    if (A.use_p2p) {  // request-sharded global alpha: sum the pair over the ranks (p2p.cuh)
        p2p_allreduce_warp(sm, stt, A.p2p, A.devstatus);
    }
    if (lane == 0) {
        ewma_apply(A.alpha, sm, stt, A.decay);
        signal_alpha_ready(A.alpha_ready);
    }
}

// One warp races max(0, p) over local columns [c0, c1) of the row at prow (c0 % 4 == 0): the R5
// fallback (emit kernels; the fused-push race epilogue for its chunk).  Returns the packed key (0: no
// positive weight).
template <bool PRUNE, bool LOGITS = false>
__device__ __forceinline__ uint64_t warp_race_cols(const RaceParams& P, const float* prow, int32_t c0, int32_t c1,
                                                int32_t sel, uint32_t rid, float M = 0.f, float inv_S = 0.f) {
    const RaceCtr rc = race_ctr((kPurposeRace << 16) | static_cast<uint32_t>(sel), rid, P.step, P.k0, P.k1);
    const int lane = threadIdx.x & 31;
    const float4* p4 = reinterpret_cast<const float4*>(prow);
    const int32_t q1 = (c1 + 3) >> 2;
    const uint32_t vbase = static_cast<uint32_t>(P.vocab_offset);
    Race F;
    F.init();
    for (int32_t f0 = c0 >> 2; f0 < q1; f0 += 32) {
        const int32_t f = f0 + lane;
        const int32_t col = 4 * f;
        float w[4] = {0.f, 0.f, 0.f, 0.f};
        uint4 r = make_uint4(0, 0, 0, 0);
        if (f < q1) {
            float4 a = p4[f];
            if (LOGITS) a = to_prob4(a, M, inv_S, P.inv_tau);
            quad_weights<true>(w, a, a, false, col, c1, -1);
            r = philox_race(rc, (vbase >> 2) + static_cast<uint32_t>(f), P);
        }
        F.quad<PRUNE>(w, r, vbase + static_cast<uint32_t>(col));
        if (PRUNE) F.sync_T();
    }
    F.finish<PRUNE>(F.T);
    return warp_max_u64(F.best);
}

// ------------------------------------------------------------------ 2. the race
// Warp-independent: every warp races work items -- (request [, position], chunk of P.chunk
// columns) -- interleaved over all warps of the grid so residual (p and q) and bonus (p
// only) rows mix on every SM.  Each step issues the loads of kUnroll float4 per lane (p,
// and q on a rejection) before racing them: one specialised Philox4x32-10 call per
// float4, the 3-instruction prune test, deferred exact evaluation of survivors.  Warps
// racing chunks of the same row share their threshold (red.max on rowT, read back before
// the final flush) and their best key (red.max on rowkey).  No barriers, no shared memory.
// One 1024-thread CTA per SM (32 warps, 64 registers): against two 512-thread CTAs per SM the race is
// 0.25 us faster (14.04 vs 14.29 us on one box) -- no second CTA whose warps the
// schedulers serve after the first's.  The alpha update then runs on the grid's item-less last warp.
#ifndef TSV_RACE_THREADS
#define TSV_RACE_THREADS 1024
#endif
#ifndef TSV_RACE_MINB
#define TSV_RACE_MINB (1024 / TSV_RACE_THREADS)
#endif
constexpr int kRaceThreads = TSV_RACE_THREADS;
constexpr int kRaceWarps = kRaceThreads / 32;
#ifndef TSV_RACE_UNROLL
#define TSV_RACE_UNROLL 2
#endif
constexpr int kUnroll = TSV_RACE_UNROLL;
#ifndef TSV_RACE_F32X2
#define TSV_RACE_F32X2 1
#endif

#ifndef TSV_TRACE
#define TSV_TRACE 0
#endif
#if TSV_TRACE
// Diagnostic builds only (-DTSV_TRACE=1, scripts/diag_trace.py): per work item, globaltimer at
// the start (after the meta load), after streaming, at the end; CTA, SM and row type.
constexpr int kTraceMax = 65536;
__device__ unsigned long long g_trace[kTraceMax][4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
#endif

__device__ __forceinline__ uint32_t nctaid_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nctaid.x;" : "=r"(r));
    return r;
}

template <int MODE, bool DENSE_Q, bool PRUNE, bool LOGITS = false, bool PUSH = false>
__global__ void __launch_bounds__(kRaceThreads, TSV_RACE_MINB) verify_race_kernel(const RaceParams P) {
    TSV_STEP_SPAN(3);
    pdl_wait();  // the scan kernel's ReqMeta / rowT / rowkey are complete and visible
    TSV_STEP_WAITED();
    pdl_launch_dependents();
    // The alpha update runs beside the race (the accepted counts are final after the scan):
    // race_update 2 -- by the grid's last warp, which has no work item (the host checked);
    // race_update 1 -- by an extra CTA 0, the first launched, when every warp has an item.
    const int32_t upd = (MODE == kLazy && P.race_update == 1) ? 1 : 0;
    if (upd && blockIdx.x == 0) {
        update_cta(P.ua);
        return;
    }
    if (MODE == kLazy && P.race_update == 2 && blockIdx.x == gridDim.x - 1 && (threadIdx.x >> 5) == kRaceWarps - 1) {
        update_warp(P.ua);
        return;
    }
    const int lane = threadIdx.x & 31;
    const int32_t warp_id = (blockIdx.x - upd) * kRaceWarps + (threadIdx.x >> 5);
    const int32_t per_req = (MODE == kLazy) ? P.n_chunks : (P.k_max + 1) * P.n_chunks;
    const int32_t n_items = P.B * per_req;
    const uint32_t vbase = static_cast<uint32_t>(P.vocab_offset);

    // the stride is re-read from %nctaid at the increment (volatile asm): kept live across the streaming
    // loop it was spilled to the stack at 64 registers
    for (int32_t item = warp_id; item < n_items; item += (static_cast<int32_t>(nctaid_x()) - upd) * kRaceWarps) {
        // request-minor order: neighbouring warps (same CTA / SM) race different requests
        const int32_t i = item % P.B;
        const int32_t rem = item / P.B;
        const int32_t c = rem % P.n_chunks;
        const int32_t j = rem / P.n_chunks;
        const ReqMeta rm = P.meta[i];
        if (rm.ok != 1) continue;
#if TSV_TRACE
        const unsigned long long tr0 = gtimer();
#endif
        const int32_t sel = (MODE == kLazy) ? rm.m : j;
        if (MODE == kShard && sel > rm.k) continue;  // no such row
        const bool residual = sel < rm.k;
        const bool use_q = DENSE_Q && residual;
        int32_t xm_local = -1;
        if (residual && !DENSE_Q) xm_local = ((MODE == kLazy) ? rm.xm : P.drafts[rm.qbase + sel]) - P.vocab_offset;
        const int32_t key_row = (MODE == kLazy) ? i : rm.r0 + sel;
        const int32_t col_begin = c * P.chunk;
        const int32_t col_end = min(P.vocab, col_begin + P.chunk);
        const float4* prow = reinterpret_cast<const float4*>(P.p + static_cast<int64_t>(rm.r0 + sel) * P.ld + col_begin);
        const float4* qrow = use_q ? reinterpret_cast<const float4*>(P.q + static_cast<int64_t>(rm.qbase + sel) * P.ld + col_begin)
                                   : prow;
        const RaceCtr rc = race_ctr((kPurposeRace << 16) | static_cast<uint32_t>(sel), rm.rid, P.step, P.k0, P.k1);
        const float4 ls = LOGITS ? P.lstats[i] : make_float4(0.f, 0.f, 0.f, 0.f);  // row m's softmax stats
        Race R;
        R.init();
        {
            // Full steps with explicit pointer / counter increments: kUnroll float4 of p (and of q on a
            // rejection) per lane per step, the Philox quad counter advancing by 32 per float4.  rem (columns
            // left in the chunk) is the loop counter and the masked tail's bound: nothing else about the chunk
            // stays live across the streaming loop (the last table)
            int32_t rem = col_end - col_begin;
            const float4* pp = prow + lane;
            const float4* qp = qrow + lane;
            uint32_t ctr = (vbase >> 2) + static_cast<uint32_t>(col_begin >> 2) + static_cast<uint32_t>(lane);
#if TSV_RACE_F32X2
            // q registers: zero for a bonus row (never loaded), so w = p - q is one unconditional FADD2
            float4 b[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) b[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#endif
            for (; rem >= 128 * kUnroll; rem -= 128 * kUnroll) {
#if TSV_RACE_F32X2
                float4 a[kUnroll];
#else
                float4 a[kUnroll], b[kUnroll];
#endif
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) a[u] = ldg_stream(pp + 32 * u);
                if (use_q) {
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) b[u] = ldg_stream(qp + 32 * u);
                }
                if (LOGITS) {  // probabilities from the logits on the fly (q only on a rejection: b stays zero)
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        a[u] = to_prob4(a[u], ls.x, ls.y, P.inv_tau);
                        if (use_q) b[u] = to_prob4(b[u], ls.z, ls.w, P.inv_tau);
                    }
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const uint32_t cu = ctr + 32u * u;
                    const uint4 r = philox_race(rc, cu, P);
#if TSV_RACE_F32X2
                    if (PRUNE && DENSE_Q) {
                        // w = p - q (FADD2 on a rejection), s = w - Tc F (FFMA2 with -Tc on both lanes)
                        uint64_t w01 = f2_pack(a[u].x, a[u].y), w23 = f2_pack(a[u].z, a[u].w);
                        w01 = f2_sub(w01, f2_pack(b[u].x, b[u].y));  // p - 0 = p exactly for a bonus row
                        w23 = f2_sub(w23, f2_pack(b[u].z, b[u].w));
                        const float2 wa = f2_unpack(w01), wb = f2_unpack(w23);
                        float w[4] = {wa.x, wa.y, wb.x, wb.y};
                        if (u == 0 && R.T == 0.0f) R.warm(w, r);
                        const uint64_t ntc = f2_pack(-R.Tc, -R.Tc);
                        const float2 sa = f2_unpack(f2_fma(ntc, f2_pack(race_F(r.x), race_F(r.y)), w01));
                        const float2 sb = f2_unpack(f2_fma(ntc, f2_pack(race_F(r.z), race_F(r.w)), w23));
                        const float sv[4] = {sa.x, sa.y, sb.x, sb.y};
                        R.quad_s(w, sv, r, cu, P.vocab_offset);
                        continue;
                    }
#endif
                    float w[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
                    race_weights<DENSE_Q>(w, b[u], use_q, residual, static_cast<int32_t>(4u * (cu - (vbase >> 2))),
                                          xm_local);
                    if (PRUNE && u == 0 && R.T == 0.0f) R.warm(w, r);
                    R.quad<PRUNE>(w, r, 4u * cu + (vbase & 3u));  // = vbase + col
                }
                if (PRUNE) R.sync_T();
                pp += 32 * kUnroll;
                qp += 32 * kUnroll;
                ctr += 32u * kUnroll;
            }
            // the rest of the chunk (< 128 kUnroll columns): one float4 per lane per step, masked at rem
            for (int32_t f0 = 0; 4 * f0 < rem; f0 += 32, pp += 32, qp += 32, ctr += 32) {
                float w[4] = {0.f, 0.f, 0.f, 0.f};
                uint4 r = make_uint4(0, 0, 0, 0);
                const int32_t cl = 4 * (f0 + lane);  // column offset inside the rest
                if (cl < rem) {
                    float4 a = ldg_stream(pp);
                    float4 b = a;
                    if (use_q) b = ldg_stream(qp);
                    if (LOGITS) {
                        a = to_prob4(a, ls.x, ls.y, P.inv_tau);
                        if (use_q) b = to_prob4(b, ls.z, ls.w, P.inv_tau);
                    }
                    w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w;
                    race_weights<DENSE_Q>(w, b, use_q, residual, static_cast<int32_t>(4u * (ctr - (vbase >> 2))),
                                          xm_local);
#pragma unroll
                    for (int e = 1; e < 4; ++e)
                        if (cl + e >= rem) w[e] = 0.0f;
                    r = philox_race(rc, ctr, P);
                }
                if (PRUNE && R.T == 0.0f) R.warm(w, r);
                R.quad<PRUNE>(w, r, 4u * ctr + (vbase & 3u));
                if (PRUNE) R.sync_T();
            }
        }
#if TSV_TRACE
        const unsigned long long tr1 = gtimer();
#endif
// TSV_ROWT_EXCHANGE=1: publish this chunk's bound to the row's slot and flush against the
// row's best bound (an L2 round trip at the end of every item); the default flushes against
// the warp's own bound -- at most one exact evaluation per lane, cheaper than the round trip
// (race 14.52 vs 14.70 us at config 2).  Results are identical either way.
#ifndef TSV_ROWT_EXCHANGE
#define TSV_ROWT_EXCHANGE 0
#endif
        if (PRUNE) {
#if TSV_ROWT_EXCHANGE
            if (lane == 0) atomicMax(P.rowT + key_row, __float_as_uint(R.T));
            const float t = __uint_as_float(*reinterpret_cast<volatile uint32_t*>(P.rowT + key_row));
            R.finish<PRUNE>(fmaxf(R.T, t));
#else
            R.finish<PRUNE>(R.T);
#endif
        }
        const uint64_t best = warp_max_u64(R.best);
        // lazy: the key row (= request i) is recomputed from the item index here rather than kept live
        // across the streaming loop (which spilled it to the stack at 64 registers)
        const int32_t key_row_end = (MODE == kLazy && !LOGITS) ? item - (item / P.B) * P.B : key_row;
        if (PUSH) {  // fused push: this chunk's key into slot [rank][c][i] of every rank
            uint64_t push = best;
            const int32_t cc = (item / P.B) % P.n_chunks;
            if (best == 0) {  // (rare; warp-uniform) the request's meta is reloaded, nothing kept live
                const ReqMeta r2 = P.meta[key_row_end];
                if (r2.m < r2.k) {
                    // no positive residual in this chunk: push its share of the R5 fallback instead (max(0,
                    // p_m) over the chunk), flagged in bit 63 (never set in a race key: scores are >= 0)
                    const int32_t cb = cc * P.chunk;
                    const uint64_t fb = warp_race_cols<PRUNE>(P, P.p + static_cast<int64_t>(r2.r0 + r2.m) * P.ld, cb,
                                                              min(P.vocab, cb + P.chunk), r2.m, r2.rid);
                    push = fb ? (fb | (1ull << 63)) : 0ull;
                }
            }
            if (lane < P.pv.G) {
                // this call's epoch (written into the request's meta by the p2p meta kernel), reloaded here
                // rather than kept live across the streaming loop
                const uint32_t push_e = __ldg(&P.meta[key_row_end].pad);
                st_ll(p2p_ckeys(P.pv, push_e, lane, P.pv.rank, cc) + key_row_end,
                      make_uint4(static_cast<uint32_t>(push), push_e, static_cast<uint32_t>(push >> 32), push_e));
            }
        } else if (lane == 0 && best) {
            atomicMax(P.rowkey + key_row_end, static_cast<unsigned long long>(best));
        }
#if TSV_TRACE
        if (lane == 0 && item < kTraceMax) {
            g_trace[item][0] = tr0;
            g_trace[item][1] = tr1;
            g_trace[item][2] = gtimer();
            g_trace[item][3] = (static_cast<unsigned long long>(blockIdx.x) << 32) | (smid() << 1) | (residual ? 1u : 0u);
        }
#endif
    }
}

// ------------------------------------------------------------------ 3. emit
// One warp per request: the row key is the red.max of every warp that raced a slice of
// the row.  A key of 0 means no element of the row had positive weight (the maximal
// element of a row is always evaluated), i.e. the residual is identically zero: the
// warp then races max(0, p_m) over the row itself (R5; measure-zero, not performance
// relevant).
template <bool PRUNE, bool LOGITS = false>
__device__ uint64_t warp_race_row(const RaceParams& P, const float* prow, int32_t sel, uint32_t rid,
                                  float M = 0.f, float inv_S = 0.f) {
    return warp_race_cols<PRUNE, LOGITS>(P, prow, 0, P.vocab, sel, rid, M, inv_S);
}

template <int MODE, bool PRUNE, bool LOGITS = false>
__device__ __forceinline__ int2 emit_unit(const RaceParams& P, int32_t unit) {  // (m, k) of a valid request
    const int lane = threadIdx.x & 31;
    if (unit >= P.B) return make_int2(-1, 0);
    // lazy: the row key is loaded next to the meta (one round trip)
    uint64_t key = (MODE == kLazy) ? P.rowkey[unit] : 0ull;
    const ReqMeta rm = P.meta[unit];
    if (rm.ok != 1) return make_int2(-1, 0);  // lazy: emitted by the scan kernel; shard: flagged by the combine
    if (MODE == kLazy) {
        if (key == 0 && rm.m < rm.k) {  // R5: residual identically zero -> race over p_m
            const float4 ls = LOGITS ? P.lstats[unit] : make_float4(0.f, 0.f, 0.f, 0.f);
            key = warp_race_row<PRUNE, LOGITS>(P, P.p + static_cast<int64_t>(rm.r0 + rm.m) * P.ld, rm.m, rm.rid,
                                               ls.x, ls.y);
        }
        // drafts x_0..x_{m-1}, the padding and num_accepted were written by the scan kernel
        if (lane == 0) {
            P.out_tokens[static_cast<int64_t>(unit) * (P.k_max + 1) + rm.m] = key ? key_index(key) : -1;
            if (!key) report(P.devstatus, TSV_DEVSTATUS_NO_WEIGHT);
        }
    } else {
        for (int32_t j = 0; j <= rm.k; ++j) {
            const int32_t row = rm.r0 + j;
            const uint64_t key = P.rowkey[row];
            uint64_t fb = 0;
            if (key == 0 && j < rm.k)  // this shard's residual is zero: its share of the R5 fallback
                fb = warp_race_row<PRUNE>(P, P.p + static_cast<int64_t>(row) * P.ld, j, rm.rid);
            if (lane == 0) {
                P.tuples[row].key = key;
                P.tuples[row].fb_key = fb;
            }
        }
    }
    return make_int2(rm.m, rm.k);
}

// UPDATE: one extra CTA (the last) runs UpdateGlobalAcceptance (Listing 1 line 19) next to
// the emitting CTAs -- the alpha update fused into the verify call.  It needs only the
// accepted counts, which the scan kernel already wrote (complete and visible here, two
// kernels back), so no inter-CTA handshake is needed.
template <int MODE, bool PRUNE, bool UPDATE, bool LOGITS = false>
__global__ void __launch_bounds__(256) verify_emit_kernel(const RaceParams P, UpdateArgs ua) {
    // TSV_VERIFY_EARLY_TRIGGER: the kernel after the call may launch while the race still runs (its
    // CTAs take the SM slots the race's tail frees); it must read nothing this call writes before its
    // own grid-dependency wait (tsv.h)
    TSV_STEP_SPAN(4);
    if (P.early_trigger) pdl_launch_dependents();
    pdl_wait();
    TSV_STEP_WAITED();
    if (!P.early_trigger) pdl_launch_dependents();
    if (UPDATE && blockIdx.x == gridDim.x - 1) {
        update_block(ua);
        return;
    }
    const int2 mk = emit_unit<MODE, PRUNE, LOGITS>(P, blockIdx.x * 8 + (threadIdx.x >> 5));
    if (MODE == kLazy && P.step_counts) add_step_counts(P.step_counts, (threadIdx.x & 31) == 0, mk.x, mk.y);
}

// ------------------------------------------------------------------------ shard combine
// One warp per request: OR the accept flags of the G shards, scan m, take the max key of
// row m over shards (fallback keys if every shard's residual was zero), emit.
__device__ __forceinline__ int2 combine_unit(const RaceParams& P, const tsv_shard_tuple* __restrict__ g, int32_t G,
                                             int32_t rows_p, int32_t i) {
    if (i >= P.B) return make_int2(-1, 0);
    const int lane = threadIdx.x & 31;
    const int32_t r0 = P.row_offsets[i];
    const int32_t r1 = P.row_offsets[i + 1];
    const int32_t k = r1 - r0 - 1;
    const int32_t qbase = r0 - i;
    const bool ok = request_rows_ok(r0, r1, i, P.k_max, rows_p, P.B);
    uint32_t flags = 0;
    bool bad = false;
    if (ok && lane < k) {
        const int32_t x = P.drafts[qbase + lane];
        bad = x < 0 || x >= P.vocab_global;
        for (int32_t s = 0; s < G; ++s) flags |= g[static_cast<int64_t>(s) * rows_p + r0 + lane].flag;
        if (!(flags & 2u)) bad = true;  // no shard owns x_j
    }
    const uint32_t badm = __ballot_sync(0xFFFFFFFFu, bad);
    const uint32_t accm = __ballot_sync(0xFFFFFFFFu, (flags & 1u) != 0);
    if (!ok || badm) {
        emit(P, i, 0, -1, -1);
        if (lane == 0) report(P.devstatus, ok ? TSV_DEVSTATUS_BAD_TOKEN : TSV_DEVSTATUS_BAD_K);
        return make_int2(-1, 0);
    }
    const uint32_t kmask = k > 0 ? ((1u << k) - 1u) : 0u;
    const uint32_t rej = ~accm & kmask;
    const int32_t m = rej ? (__ffs(rej) - 1) : k;
    uint64_t key = 0, fb = 0;
    for (int32_t s = lane; s < G; s += 32) {
        const tsv_shard_tuple t = g[static_cast<int64_t>(s) * rows_p + r0 + m];
        key = t.key > key ? t.key : key;
        fb = t.fb_key > fb ? t.fb_key : fb;
    }
    key = warp_max_u64(key);
    fb = warp_max_u64(fb);
    if (key == 0 && m < k) key = fb;
    emit(P, i, qbase, m, key ? key_index(key) : -1);
    if (lane == 0 && !key) report(P.devstatus, TSV_DEVSTATUS_NO_WEIGHT);
    return make_int2(m, k);
}

__global__ void verify_shard_combine_kernel(const RaceParams P, const tsv_shard_tuple* __restrict__ g,
                                            int32_t G, int32_t rows_p) {
    pdl_wait();
    pdl_launch_dependents();
    const int32_t i = blockIdx.x * static_cast<int32_t>(blockDim.x >> 5) + static_cast<int32_t>(threadIdx.x >> 5);
    const int2 mk = combine_unit(P, g, G, rows_p, i);
    if (P.step_counts) add_step_counts(P.step_counts, (threadIdx.x & 31) == 0, mk.x, mk.y);
}

// ------------------------------------------------------------ lazy two-round vocab sharding
// Round 1 (flags): per request, the accept and owner bits of the drafts this shard owns;
// ownership is disjoint across shards, so the integer sum of the G mask words is their OR.
// Round 2 (race): from the summed masks every shard forms the same m_i, races row m_i over
// its columns and publishes (local key, local fallback key); the element-wise max over
// shards is the unsharded row key.  Emit: from summed masks + maxed keys.
// Warp-collective: the request's mask word (owner bits << 32 | accept bits) on this shard.
__device__ __forceinline__ unsigned long long shard_flags_mask(const RaceParams& P, int32_t i) {
    const int lane = threadIdx.x & 31;
    const int32_t r0 = P.row_offsets[i];
    const int32_t r1 = P.row_offsets[i + 1];
    const int32_t k = r1 - r0 - 1;
    const int32_t qbase = r0 - i;
    const bool ok = request_rows_ok(r0, r1, i, P.k_max, P.rows_p, P.B);
    bool acc = false, own = false;
    if (ok && lane < k) {
        const int32_t x = P.drafts[qbase + lane];
        const int32_t xl = x - P.vocab_offset;
        own = x >= 0 && x < P.vocab_global && xl >= 0 && xl < P.vocab;
        if (own) {
            const uint32_t rid = P.rids[i];
            const uint4 rr = philox4x32_10(0u, (kPurposeAccept << 16) | static_cast<uint32_t>(lane), rid, P.step,
                                           P.k0, P.k1);
            const float u = u_acc_from_word(rr.x);
            const float qx = P.q ? P.q[static_cast<int64_t>(qbase + lane) * P.ld + xl] : 1.0f;
            const float px = P.p[static_cast<int64_t>(r0 + lane) * P.ld + xl];
            acc = __fmul_rn(u, qx) < px;  // strict; NaN rejects
        }
    }
    const uint32_t accm = __ballot_sync(0xFFFFFFFFu, acc);
    const uint32_t ownm = __ballot_sync(0xFFFFFFFFu, own);
    return (static_cast<unsigned long long>(ownm) << 32) | accm;
}

__global__ void __launch_bounds__(256) verify_shard_flags_kernel(const RaceParams P, unsigned long long* masks) {
    pdl_wait();
    pdl_launch_dependents();
    zero_step_counts(P.step_counts);
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const unsigned long long mask = shard_flags_mask(P, i);
    if ((threadIdx.x & 31) == 0) masks[i] = mask;
}

// The request's ReqMeta from the summed mask word (every lane; identical on every shard).
// ok: 1 valid, 0 bad k, 2 bad draft (outside [0, vocab_global) or owned by no shard).
__device__ __forceinline__ ReqMeta shard_meta_from_masks(const RaceParams& P, int32_t i, unsigned long long mask) {
    const int lane = threadIdx.x & 31;
    const int32_t r0 = P.row_offsets[i];
    const int32_t r1 = P.row_offsets[i + 1];
    const int32_t k = r1 - r0 - 1;
    const int32_t qbase = r0 - i;
    int32_t ok = request_rows_ok(r0, r1, i, P.k_max, P.rows_p, P.B) ? 1 : 0;
    int32_t x = -1;
    bool bad = false;
    if (ok && lane < k) {
        x = P.drafts[qbase + lane];
        bad = x < 0 || x >= P.vocab_global;
    }
    const uint32_t accm = static_cast<uint32_t>(mask);
    const uint32_t ownm = static_cast<uint32_t>(mask >> 32);
    const uint32_t kmask = (ok == 1 && k > 0) ? ((1u << k) - 1u) : 0u;
    if (__ballot_sync(0xFFFFFFFFu, bad) || (ownm & kmask) != kmask) ok = ok ? 2 : 0;
    const uint32_t rej = ~accm & kmask;
    const int32_t m = ok == 1 ? (rej ? (__ffs(rej) - 1) : k) : -1;
    const int32_t xm = __shfl_sync(0xFFFFFFFFu, x, (m >= 0 ? m : 0) & 31);
    ReqMeta rm;
    rm.r0 = r0;
    rm.k = k;
    rm.qbase = qbase;
    rm.m = m;
    rm.xm = (m >= 0 && m < k) ? xm : -1;
    rm.ok = ok;
    rm.rid = P.rids[i];
    rm.pad = 0;
    return rm;
}

__global__ void __launch_bounds__(256) verify_shard_meta_kernel(const RaceParams P, const unsigned long long* masks) {
    pdl_wait();
    pdl_launch_dependents();
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const ReqMeta rm = shard_meta_from_masks(P, i, masks[i]);
    if ((threadIdx.x & 31) == 0) {
        P.meta[i] = rm;
        P.rowT[i] = 0u;
        P.rowkey[i] = 0ull;
    }
}

template <bool PRUNE>
__global__ void __launch_bounds__(256) verify_shard_keys_kernel(const RaceParams P, unsigned long long* keys) {
    pdl_wait();
    pdl_launch_dependents();
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const int lane = threadIdx.x & 31;
    const ReqMeta rm = P.meta[i];
    uint64_t key = 0, fb = 0;
    if (rm.ok == 1) {
        key = P.rowkey[i];
        if (key == 0 && rm.m < rm.k)  // this shard's residual is zero: its share of the R5 fallback
            fb = warp_race_row<PRUNE>(P, P.p + static_cast<int64_t>(rm.r0 + rm.m) * P.ld, rm.m, rm.rid);
    }
    if (lane == 0) {
        keys[2 * i] = key;
        keys[2 * i + 1] = fb;
    }
}

__device__ __forceinline__ int2 shard_emit_unit(const RaceParams& P, const unsigned long long* masks,
                                                const unsigned long long* keys, int32_t i) {
    if (i >= P.B) return make_int2(-1, 0);
    const int lane = threadIdx.x & 31;
    const ReqMeta rm = shard_meta_from_masks(P, i, masks[i]);
    if (rm.ok != 1) {
        emit(P, i, 0, -1, -1);
        if (lane == 0) report(P.devstatus, rm.ok == 2 ? TSV_DEVSTATUS_BAD_TOKEN : TSV_DEVSTATUS_BAD_K);
        return make_int2(-1, 0);
    }
    uint64_t key = keys[2 * i];
    if (key == 0 && rm.m < rm.k) key = keys[2 * i + 1];
    emit(P, i, rm.qbase, rm.m, key ? key_index(key) : -1);
    if (lane == 0 && !key) report(P.devstatus, TSV_DEVSTATUS_NO_WEIGHT);
    return make_int2(rm.m, rm.k);
}

__global__ void __launch_bounds__(256) verify_shard_emit_kernel(const RaceParams P, const unsigned long long* masks,
                                                                const unsigned long long* keys) {
    pdl_wait();
    pdl_launch_dependents();
    const int2 mk = shard_emit_unit(P, masks, keys, blockIdx.x * 8 + (threadIdx.x >> 5));
    if (P.step_counts) add_step_counts(P.step_counts, (threadIdx.x & 31) == 0, mk.x, mk.y);
}

// ------------------------------------------------ vocab sharding over peer memory (NEXT 3)
// The lazy two rounds with the two exchanges done by the producing kernels themselves over
// NVLink peer memory instead of NCCL all-reduces.  Every rank owns
// one symmetric buffer, mapped into every peer (CUDA IPC).  Each exchanged 32-bit word
// travels with the call's epoch in one 8-byte word {data, epoch} (the "LL" idea: an
// aligned 8-byte store arrives whole), written with 16-byte vector stores into slot
// [rank][i] of every peer's buffer.  The consumer of request i polls its own buffer's G
// slots until every word carries the epoch -- no fences, no grid barrier, no flag round
// trip -- and combines: the sum of the disjoint mask words (round 1, flags -> meta), the max
// of the packed keys (round 2, keys -> emit).  Slots alternate by epoch parity.  The epoch
// lives on the device (own buffer), read by every kernel of a call and advanced by the
// emit kernel's last CTA, so captured CUDA graphs replay with advancing epochs.  A wait
// gives up after seconds and sets TSV_DEVSTATUS_P2P_TIMEOUT instead of hanging.
// All-reduce (sum) of count <= TSV_P2P_MAX_SUMS int64 over the ranks (request-sharded global
// goodput / acceptance sums, p2p.cuh): one CTA, data in global memory.
__global__ void __launch_bounds__(64) p2p_allreduce_i64_kernel(int64_t* data, int32_t count, const P2PView V,
                                                               int32_t* devstatus) {
    pdl_wait();
    pdl_launch_dependents();
    p2p_allreduce_block(reinterpret_cast<long long*>(data), count, V, devstatus);
}

// NC > 0 (fused push): this rank races P.n_chunks <= NC chunks per row; the slots of chunks
// P.n_chunks .. NC-1 (uneven shards) get an empty key here, so every rank's emit polls NC slots per rank.
__global__ void __launch_bounds__(256) verify_p2p_flags_kernel(const RaceParams P, const P2PView V, int32_t NC) {
    pdl_wait();
    pdl_launch_dependents();
    zero_step_counts(P.step_counts);
    const uint32_t e = p2p_load_epoch(V);
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const unsigned long long mask = shard_flags_mask(P, i);
    const int lane = threadIdx.x & 31;
    if (lane < V.G)  // lane g stores into rank g's buffer
        st_ll(p2p_masks(V, e, lane, V.rank) + i,
              make_uint4(static_cast<uint32_t>(mask), e, static_cast<uint32_t>(mask >> 32), e));
    for (int32_t idx = lane; idx < V.G * (NC - P.n_chunks); idx += 32)
        st_ll(p2p_ckeys(V, e, idx % V.G, V.rank, P.n_chunks + idx / V.G) + i, make_uint4(0u, e, 0u, e));
}

__global__ void __launch_bounds__(256) verify_p2p_meta_kernel(const RaceParams P, const P2PView V) {
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t e = p2p_load_epoch(V);
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const int lane = threadIdx.x & 31;
    unsigned long long mask = 0;  // lane g polls rank g's words; disjoint owners: the sum is the OR
    if (lane < V.G) {
        const uint4 v = ld_ll_wait(p2p_masks(V, e, V.rank, lane) + i, e, P.devstatus);
        mask = (static_cast<unsigned long long>(v.z) << 32) | v.x;
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) mask += __shfl_xor_sync(0xFFFFFFFFu, mask, o);  // lanes 0..7
    mask = __shfl_sync(0xFFFFFFFFu, mask, 0);
    ReqMeta rm = shard_meta_from_masks(P, i, mask);
    rm.pad = e;  // the call's epoch, for the fused-push race items (no epoch load in the race kernel)
    if (lane == 0) {
        P.meta[i] = rm;
        P.rowT[i] = 0u;
        P.rowkey[i] = 0ull;
    }
}

template <bool PRUNE>
__global__ void __launch_bounds__(256) verify_p2p_keys_kernel(const RaceParams P, const P2PView V) {
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t e = p2p_load_epoch(V);
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const int lane = threadIdx.x & 31;
    const ReqMeta rm = P.meta[i];
    uint64_t key = 0, fb = 0;
    if (rm.ok == 1) {
        key = P.rowkey[i];
        if (key == 0 && rm.m < rm.k)  // this shard's residual is zero: its share of the R5 fallback
            fb = warp_race_row<PRUNE>(P, P.p + static_cast<int64_t>(rm.r0 + rm.m) * P.ld, rm.m, rm.rid);
    }
    if (lane < V.G) {
        uint4* d = p2p_keys(V, e, lane, V.rank) + 2 * i;
        st_ll(d, make_uint4(static_cast<uint32_t>(key), e, static_cast<uint32_t>(key >> 32), e));
        st_ll(d + 1, make_uint4(static_cast<uint32_t>(fb), e, static_cast<uint32_t>(fb >> 32), e));
    }
}

__global__ void __launch_bounds__(256) verify_p2p_emit_kernel(const RaceParams P, const P2PView V) {
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t e = p2p_load_epoch(V);
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    int2 mk = make_int2(-1, 0);
    if (i < P.B) {
        const int lane = threadIdx.x & 31;
        const ReqMeta rm = P.meta[i];  // written by this rank's meta kernel (same m_i on every rank)
        uint64_t key = 0, fb = 0;
        if (lane < V.G) {  // poll every rank's words (also for bad requests: keeps the slots' epochs in step)
            const uint4* s = p2p_keys(V, e, V.rank, lane) + 2 * i;
            const uint4 a = ld_ll_wait(s, e, P.devstatus);
            const uint4 b = ld_ll_wait(s + 1, e, P.devstatus);
            key = (static_cast<uint64_t>(a.z) << 32) | a.x;
            fb = (static_cast<uint64_t>(b.z) << 32) | b.x;
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            const uint64_t k2 = __shfl_xor_sync(0xFFFFFFFFu, key, o), f2 = __shfl_xor_sync(0xFFFFFFFFu, fb, o);
            key = k2 > key ? k2 : key;
            fb = f2 > fb ? f2 : fb;
        }
        key = __shfl_sync(0xFFFFFFFFu, key, 0);
        fb = __shfl_sync(0xFFFFFFFFu, fb, 0);
        if (rm.ok != 1) {
            emit(P, i, 0, -1, -1);
            if (lane == 0) report(P.devstatus, rm.ok == 2 ? TSV_DEVSTATUS_BAD_TOKEN : TSV_DEVSTATUS_BAD_K);
        } else {
            if (key == 0 && rm.m < rm.k) key = fb;
            emit(P, i, rm.qbase, rm.m, key ? key_index(key) : -1);
            if (lane == 0 && !key) report(P.devstatus, TSV_DEVSTATUS_NO_WEIGHT);
            mk = make_int2(rm.m, rm.k);
        }
    }
    if (P.step_counts) add_step_counts(P.step_counts, (threadIdx.x & 31) == 0, mk.x, mk.y);
    // advance the device epoch once every CTA of this kernel has read it (last CTA, GPU scope)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p2p_counter(V), 1u) == gridDim.x - 1) {
            atomicExch(p2p_counter(V), 0u);
            atomicExch(p2p_epoch(V), e);
        }
    }
}

// Fused-push emit (TSV_VERIFY_P2P_FUSED): the race items pushed their chunk keys as LL lines, so
// request i's warp polls the G x NC lines of its own buffer (lane-strided), takes the max and emits;
// no keys kernel.  A race item whose chunk has no positive residual pushed its chunk's share of the R5
// fallback instead, flagged in bit 63: the max of the flagged keys is used only when every chunk of
// every rank had a zero residual (R5), exactly the fallback of the unsharded verify.
template <bool PRUNE>
__global__ void __launch_bounds__(256) verify_p2p_emit_push_kernel(const RaceParams P, const P2PView V, int32_t NC) {
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t e = p2p_load_epoch(V);
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    int2 mk = make_int2(-1, 0);
    if (i < P.B) {
        const int lane = threadIdx.x & 31;
        const ReqMeta rm = P.meta[i];  // same m_i on every rank
        if (rm.ok != 1) {
            emit(P, i, 0, -1, -1);
            if (lane == 0) report(P.devstatus, rm.ok == 2 ? TSV_DEVSTATUS_BAD_TOKEN : TSV_DEVSTATUS_BAD_K);
        } else {
            uint64_t key = 0, fb = 0;  // max race key; max flagged chunk fallback key (bit 63)
            for (int32_t idx = lane; idx < V.G * NC; idx += 32) {
                const uint4 v = ld_ll_wait(p2p_ckeys(V, e, V.rank, idx / NC, idx % NC) + i, e, P.devstatus);
                const uint64_t k = (static_cast<uint64_t>(v.z) << 32) | v.x;
                if (k >> 63) {
                    const uint64_t f = k & ~(1ull << 63);
                    fb = f > fb ? f : fb;
                } else {
                    key = k > key ? k : key;
                }
            }
            key = warp_max_u64(key);
            fb = warp_max_u64(fb);
            if (key == 0 && rm.m < rm.k) key = fb;  // R5: the residual is zero on every rank
            emit(P, i, rm.qbase, rm.m, key ? key_index(key) : -1);
            if (lane == 0 && !key) report(P.devstatus, TSV_DEVSTATUS_NO_WEIGHT);
            mk = make_int2(rm.m, rm.k);
        }
    }
    if (P.step_counts) add_step_counts(P.step_counts, (threadIdx.x & 31) == 0, mk.x, mk.y);
    // advance the device epoch once every CTA of this kernel has read it (last CTA, GPU scope)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p2p_counter(V), 1u) == gridDim.x - 1) {
            atomicExch(p2p_counter(V), 0u);
            atomicExch(p2p_epoch(V), e);
        }
    }
}

// ------------------------------------------------------------------ greedy verify (NEXT 2)
__global__ void __launch_bounds__(256) clear_u64_kernel(unsigned long long* p, int64_t n, long long* step_counts) {
    pdl_wait();  // the previous call's readers of these slots are done
    pdl_launch_dependents();
    zero_step_counts(step_counts);
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 1024 + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (i0 + 256 * k < n) p[i0 + 256 * k] = 0ull;
}

// Temperature 0 (reading R24): keep draft j iff x_j = argmax_v p_j[v]; emit the argmax of
// row m.  Every row up to the first mismatch needs its full argmax, so the rows are streamed
// densely: work items (row, chunk) grid-stride over all p rows of the batch; a lane keeps its
// first maximum (strict >, NaN never selected), the warp combines packed keys
// (monotone(value) << 32 | ~v: max value, then lowest index) and red.max-es them into the
// row's slot; one warp per request then scans for the first mismatch and emits.
__device__ __forceinline__ uint64_t greedy_key(float f, int32_t v) {  // v < 0: none
    if (v < 0) return 0ull;
    uint32_t u = __float_as_uint(f == 0.0f ? 0.0f : f);  // +0 == -0
    u = (u >> 31) ? ~u : (u | 0x80000000u);               // order-preserving for non-NaN floats
    return (static_cast<uint64_t>(u) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(v));
}

#ifndef TSV_GREEDY_MINB
#define TSV_GREEDY_MINB 8  // 64 warps per SM: 32.2 us vs 44.3 us at 32 (config 2)
#endif
__global__ void __launch_bounds__(256, TSV_GREEDY_MINB) verify_greedy_argmax_kernel(const RaceParams P) {
    pdl_wait();
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int32_t warp_id = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int32_t n_warps = gridDim.x * 8;
    const int32_t rows = dense_rows(P.row_offsets, P.B, P.rows_p);  // p rows that belong to requests
    const int64_t n_items = static_cast<int64_t>(rows) * P.n_chunks;
    for (int64_t item = warp_id; item < n_items; item += n_warps) {
        const int32_t r = static_cast<int32_t>(item % rows);  // row-minor: neighbours stream different rows
        const int32_t c = static_cast<int32_t>(item / rows);
        const int32_t col_begin = c * P.chunk;
        const int32_t col_end = min(P.vocab, col_begin + P.chunk);
        const float4* prow = reinterpret_cast<const float4*>(P.p + static_cast<int64_t>(r) * P.ld + col_begin);
        const int32_t nq = (col_end - col_begin + 3) >> 2;
        const int32_t nq_full = (col_end - col_begin) >> 2;  // float4s entirely inside the row
        float best_f = 0.0f;
        int32_t best_v = -1;
        auto take = [&](float f, int32_t v) {
            if (f == f && (best_v < 0 || f > best_f)) {
                best_f = f;
                best_v = v;
            }
        };
#ifndef TSV_GREEDY_UNROLL
#define TSV_GREEDY_UNROLL 3
#endif
        constexpr int GU = TSV_GREEDY_UNROLL;  // float4 per lane in flight (config 2: 3 -> 29.2 us; 2: 30.0; 4: 30.7, spills)
        int32_t f = lane;
        for (; f + 32 * (GU - 1) < nq_full; f += 32 * GU) {
            float4 a[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u) a[u] = ldg_stream(prow + f + 32 * u);
            const int32_t v = col_begin + 4 * f;
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                take(a[u].x, v + 128 * u);
                take(a[u].y, v + 128 * u + 1);
                take(a[u].z, v + 128 * u + 2);
                take(a[u].w, v + 128 * u + 3);
            }
        }
        for (; f < nq; f += 32) {
            const float4 a = ldg_stream(prow + f);
            const int32_t v = col_begin + 4 * f;
            const float e[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (v + t < col_end) take(e[t], v + t);
        }
        const uint64_t key = warp_max_u64(greedy_key(best_f, best_v));
        if (lane == 0 && key) atomicMax(P.rowkey + r, static_cast<unsigned long long>(key));
    }
}

__device__ __forceinline__ int2 greedy_emit_unit(const RaceParams& P, int32_t i) {
    if (i >= P.B) return make_int2(-1, 0);
    const int lane = threadIdx.x & 31;
    const int32_t r0 = P.row_offsets[i];
    const int32_t r1 = P.row_offsets[i + 1];
    const int32_t k = r1 - r0 - 1;
    const int32_t qbase = r0 - i;
    const bool ok = request_rows_ok(r0, r1, i, P.k_max, dense_rows(P.row_offsets, P.B, P.rows_p), P.B);
    int32_t x = -1, g = -1;
    bool bad = false;
    if (ok && lane <= k) {
        const uint64_t key = P.rowkey[r0 + lane];
        g = key ? key_index(key) : -1;
        if (lane < k) {
            x = P.drafts[qbase + lane];
            bad = x < 0 || x >= P.vocab;
        }
    }
    if (!ok || __ballot_sync(0xFFFFFFFFu, bad)) {
        emit(P, i, 0, -1, -1);
        if (lane == 0) report(P.devstatus, ok ? TSV_DEVSTATUS_BAD_TOKEN : TSV_DEVSTATUS_BAD_K);
        return make_int2(-1, 0);
    }
    const uint32_t mism = __ballot_sync(0xFFFFFFFFu, lane < k && x != g);
    const int32_t m = mism ? __ffs(mism) - 1 : k;
    const int32_t t = __shfl_sync(0xFFFFFFFFu, g, m);
    emit(P, i, qbase, m, t);
    if (lane == 0 && t < 0) report(P.devstatus, TSV_DEVSTATUS_NO_WEIGHT);
    return make_int2(m, k);
}

__global__ void __launch_bounds__(256) verify_greedy_emit_kernel(const RaceParams P) {
    pdl_wait();
    pdl_launch_dependents();
    const int2 mk = greedy_emit_unit(P, blockIdx.x * 8 + (threadIdx.x >> 5));
    if (P.step_counts) add_step_counts(P.step_counts, (threadIdx.x & 31) == 0, mk.x, mk.y);
}

// ------------------------------------------------------------ fused softmax from logits (NEXT 1)
// p and q arrive as logits (reading R23).  Pass 1 (dense, every p and q row of the batch):
// per (row, chunk) item the warp's online softmax partial (m_c = max z, s_c = sum of
// expf((z - m_c) / tau) in binary64) goes to a partials table.  Pass 2 (one warp per
// request): lanes combine the partials of rows j (M = max m_c, S = sum s_c exp((m_c - M)/tau)),
// run the acceptance test on p_j[x_j], q_j[x_j] computed from the logits, and publish
// row m's (M_p, 1/S_p, M_q, 1/S_q) next to ReqMeta.  Then the lazy race streams row m's logits
// and forms the probabilities on the fly -- p and q are never written out.
struct LogitPartial {
    float m;
    float pad;
    double s;
};

__device__ __forceinline__ uint32_t ordered_bits(float f) {  // monotone float -> uint (no NaN)
    const uint32_t u = __float_as_uint(f);
    return (u >> 31) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float from_ordered_bits(uint32_t k) {
    return __uint_as_float((k >> 31) ? (k & 0x7FFFFFFFu) : ~k);
}
__device__ __forceinline__ float exp_arg(float z, float m, float inv_tau) {
    return __fmul_rn(__fsub_rn(z, m), inv_tau);
}
// Terms of the row sums only (never a probability): 2^(RN32(z - m) * RN32(log2(e) / tau)) by one
// MUFU.EX2 (ex2.approx, relative error ~2^-22, the same order as expf's 2 ulp; results below
// 2^-126 flush to 0, which a sum >= 1 in binary64 cannot see).  The probabilities themselves
// (to_prob: scan gathers, the race, softmax rows) keep the accurate expf.
#ifndef TSV_STATS_FAST_EXP
#define TSV_STATS_FAST_EXP 1
#endif
__device__ __forceinline__ float sum_term(float z, float m, float inv_tau, float l2e_tau) {
#if TSV_STATS_FAST_EXP
    (void)inv_tau;
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fmul_rn(__fsub_rn(z, m), l2e_tau)));
    return r;
#else
    (void)l2e_tau;
    return expf(exp_arg(z, m, inv_tau));
#endif
}

// Pass 1: per (row, chunk) item, a warp-uniform running max m (raised at most once per step
// for all lanes -- no divergent rescaling) and per-lane sums of expf((z - m) / tau): four
// exponentials added in fp32, then accumulated in binary64.  Stored as (m, sum).
#ifndef TSV_STATS_MINB
#define TSV_STATS_MINB 4
#endif
__global__ void __launch_bounds__(256, TSV_STATS_MINB) verify_logit_stats_kernel(const RaceParams P, LogitPartial* part,
                                                                    int32_t rows_q_max) {
    pdl_wait();
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int32_t warp_id = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int32_t n_warps = gridDim.x * 8;
    const int32_t rp = dense_rows(P.row_offsets, P.B, P.rows_p);  // p rows in use; q rows: rp - B
    const int32_t rq = (P.q != nullptr) ? max(0, min(rp - P.B, rows_q_max)) : 0;
    const int64_t n_items = static_cast<int64_t>(rp + rq) * P.n_chunks;
    const float it = P.inv_tau;
    const float l2e = __fmul_rn(1.4426950408889634f, it);  // RN32(log2(e) / tau)
    for (int64_t item = warp_id; item < n_items; item += n_warps) {
        const int32_t r = static_cast<int32_t>(item % (rp + rq));
        const int32_t c = static_cast<int32_t>(item / (rp + rq));
        const bool isq = r >= rp;
        const float* row = isq ? P.q + static_cast<int64_t>(r - rp) * P.ld : P.p + static_cast<int64_t>(r) * P.ld;
        const int32_t col_begin = c * P.chunk;
        const int32_t col_end = min(P.vocab, col_begin + P.chunk);
        const float4* z4 = reinterpret_cast<const float4*>(row + col_begin);
        const int32_t nq = (col_end - col_begin + 3) >> 2;
        float m = -INFINITY;
        double s = 0.0;
#ifndef TSV_STATS_U
#define TSV_STATS_U 4
#endif
        constexpr int SU = TSV_STATS_U;  // float4 per lane per step
        auto load2 = [&](int32_t f0, float4 (&z)[SU]) {
#pragma unroll
            for (int h = 0; h < SU; ++h) {
                const int32_t f = f0 + 32 * h + lane;
                z[h] = f < nq ? ldg_stream(z4 + f) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
        };
        float4 cur[SU];
        load2(0, cur);
        for (int32_t f0 = 0; f0 < nq; f0 += 32 * SU) {  // SU float4 per lane; the next SU in flight
            float4 nxt[SU];
            if (f0 + 32 * SU < nq) load2(f0 + 32 * SU, nxt);
            float e[4 * SU];
#pragma unroll
            for (int h = 0; h < SU; ++h) {
                const int32_t v = col_begin + 4 * (f0 + 32 * h + lane);
                e[4 * h + 0] = cur[h].x;
                e[4 * h + 1] = v + 1 < col_end ? cur[h].y : -INFINITY;
                e[4 * h + 2] = v + 2 < col_end ? cur[h].z : -INFINITY;
                e[4 * h + 3] = v + 3 < col_end ? cur[h].w : -INFINITY;
            }
            float lm = e[0];
#pragma unroll
            for (int t = 1; t < 4 * SU; ++t) lm = fmaxf(lm, e[t]);
            const float wm = from_ordered_bits(__reduce_max_sync(0xFFFFFFFFu, ordered_bits(lm)));
            if (wm > m) {  // warp-uniform
                if (m > -INFINITY) s *= static_cast<double>(expf(exp_arg(m, wm, it)));
                m = wm;
            }
            float acc = 0.0f;
#pragma unroll
            for (int h = 0; h < SU; ++h) {
                float x[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) x[t] = e[4 * h + t] > -INFINITY ? sum_term(e[4 * h + t], m, it, l2e) : 0.0f;
                acc = __fadd_rn(acc, __fadd_rn(__fadd_rn(x[0], x[1]), __fadd_rn(x[2], x[3])));
            }
            s += static_cast<double>(acc);
#pragma unroll
            for (int h = 0; h < SU; ++h) cur[h] = nxt[h];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        if (lane == 0) {
            const int64_t slot = (isq ? static_cast<int64_t>(P.rows_p) + (r - rp) : r) * P.n_chunks + c;
            part[slot].m = m;
            part[slot].pad = 0.f;
            part[slot].s = s;
        }
    }
}

// (M, RN32(1/S)) of one row from its chunk partials.
__device__ __forceinline__ float2 logit_row_stats(const RaceParams& P, const LogitPartial* part, int64_t slot0) {
    float M = -INFINITY;
    for (int32_t c = 0; c < P.n_chunks; ++c) M = fmaxf(M, part[slot0 + c].m);
    double S = 0.0;
    for (int32_t c = 0; c < P.n_chunks; ++c) {
        const LogitPartial pc = part[slot0 + c];
        if (pc.m > -INFINITY) S += pc.s * static_cast<double>(expf(exp_arg(pc.m, M, P.inv_tau)));
    }
    return make_float2(M, __double2float_rn(1.0 / S));
}

__global__ void __launch_bounds__(256) verify_logit_scan_kernel(const RaceParams P, const LogitPartial* part,
                                                                float4* lstats) {
    pdl_wait();
    pdl_launch_dependents();
    zero_step_counts(P.step_counts);
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const int lane = threadIdx.x & 31;
    const int32_t r0 = P.row_offsets[i];
    const int32_t r1 = P.row_offsets[i + 1];
    const int32_t k = r1 - r0 - 1;
    const int32_t qbase = r0 - i;
    int32_t ok = request_rows_ok(r0, r1, i, P.k_max, dense_rows(P.row_offsets, P.B, P.rows_p), P.B) ? 1 : 0;
    const uint32_t rid = P.rids[i];
    int32_t x = -1;
    bool bad = false, acc = false;
    float2 sp = make_float2(0.f, 0.f), sq = make_float2(0.f, 0.f);
    if (ok && lane <= k) sp = logit_row_stats(P, part, static_cast<int64_t>(r0 + lane) * P.n_chunks);
    if (ok && lane < k && P.q) sq = logit_row_stats(P, part, (static_cast<int64_t>(P.rows_p) + qbase + lane) * P.n_chunks);
    if (ok && lane < k) {
        x = P.drafts[qbase + lane];
        bad = x < 0 || x >= P.vocab;
        if (!bad) {
            const uint4 rr = philox4x32_10(0u, (kPurposeAccept << 16) | static_cast<uint32_t>(lane), rid, P.step,
                                           P.k0, P.k1);
            const float u = u_acc_from_word(rr.x);
            const float qx = P.q ? to_prob(P.q[static_cast<int64_t>(qbase + lane) * P.ld + x], sq.x, sq.y, P.inv_tau) : 1.0f;
            const float px = to_prob(P.p[static_cast<int64_t>(r0 + lane) * P.ld + x], sp.x, sp.y, P.inv_tau);
            acc = __fmul_rn(u, qx) < px;  // strict; NaN rejects
        }
    }
    if (__ballot_sync(0xFFFFFFFFu, bad)) ok = 2;
    const uint32_t accm = __ballot_sync(0xFFFFFFFFu, acc);
    const uint32_t kmask = (ok == 1 && k > 0) ? ((1u << k) - 1u) : 0u;
    const uint32_t rej = ~accm & kmask;
    const int32_t m = rej ? (__ffs(rej) - 1) : (ok == 1 ? k : -1);
    const int32_t src = (m >= 0 ? m : 0) & 31;
    const int32_t xm = __shfl_sync(0xFFFFFFFFu, x, src);
    const float4 st = make_float4(__shfl_sync(0xFFFFFFFFu, sp.x, src), __shfl_sync(0xFFFFFFFFu, sp.y, src),
                                  __shfl_sync(0xFFFFFFFFu, sq.x, src), __shfl_sync(0xFFFFFFFFu, sq.y, src));
    if (lane == 0) {
        ReqMeta rm;
        rm.r0 = r0;
        rm.k = k;
        rm.qbase = qbase;
        rm.m = m;
        rm.xm = (m >= 0 && m < k) ? xm : -1;
        rm.ok = ok;
        rm.rid = rid;
        rm.pad = 0;
        P.meta[i] = rm;
        lstats[i] = st;
        P.rowT[i] = 0u;
        P.rowkey[i] = 0ull;
        P.num_accepted[i] = m;
    }
    if (ok == 1) emit_prefix(P, i, m, x);
    else {
        emit(P, i, 0, -1, -1);
        if (lane == 0) report(P.devstatus, ok == 2 ? TSV_DEVSTATUS_BAD_TOKEN : TSV_DEVSTATUS_BAD_K);
    }
}

// Standalone softmax rows (reading R23), one CTA per row: max, binary64 sum of expf, write p.
__global__ void __launch_bounds__(256) softmax_rows_kernel(const float* z, int64_t ld, int32_t V, float inv_tau,
                                                           float* out) {
    __shared__ float s_m[8];
    __shared__ double s_s[8];
    pdl_wait();
    pdl_launch_dependents();
    const float* zr = z + static_cast<int64_t>(blockIdx.x) * ld;
    float* pr = out + static_cast<int64_t>(blockIdx.x) * ld;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float m = -INFINITY;
    for (int32_t v = threadIdx.x; v < V; v += 256) m = fmaxf(m, zr[v]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if (lane == 0) s_m[warp] = m;
    __syncthreads();
    float M = s_m[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) M = fmaxf(M, s_m[w]);
    double s = 0.0;  // the row sum with the terms of the verify's statistics pass (sum_term)
    const float l2e = __fmul_rn(1.4426950408889634f, inv_tau);
    for (int32_t v = threadIdx.x; v < V; v += 256)
        if (zr[v] > -INFINITY) s += static_cast<double>(sum_term(zr[v], M, inv_tau, l2e));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if (lane == 0) s_s[warp] = s;
    __syncthreads();
    double S = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) S += s_s[w];
    const float inv_S = __double2float_rn(1.0 / S);
    for (int32_t v = threadIdx.x; v < V; v += 256) pr[v] = to_prob(zr[v], M, inv_S, inv_tau);
    for (int64_t v = V + threadIdx.x; v < ld; v += 256) pr[v] = 0.0f;
}

// ------------------------------------------------------------------------ host side
static int sm_count();
// Default work-item size: about one item per resident warp of the race kernel
// (148 SMs x 4 CTAs x 8 warps), in whole 128-column iterations.  Never changes results.
static int32_t auto_chunk(const tsv_verify_args* a) {
    if (a->chunk > 0) return a->chunk;
    const int64_t warps = static_cast<int64_t>(sm_count()) * kRaceWarps * TSV_RACE_MINB;  // resident race warps
    // chunks per row so that B * chunks <= warps (one wave), then the chunk covering V in that many
    const int64_t per_row = std::max<int64_t>(1, warps / std::max<int32_t>(a->B, 1));
    int64_t c = (a->vocab + per_row - 1) / per_row;
    c = (c + 127) / 128 * 128;
    if (c < 512) c = 512;
    if (c > kMaxChunk) c = kMaxChunk;
    return static_cast<int32_t>(c);
}

// Fused push (TSV_VERIFY_P2P_FUSED): every rank must agree on NC, the number of chunk slots per row
// and rank, from what all ranks know (vocab_global, the world size, B, the SM count): chunks sized as
// auto_chunk would for the largest shard ceil4(vocab_global / G), at most kP2PMaxChunks of them.
// This rank races ceil(vocab / chunk) <= NC chunks (its shard may be smaller).
static tsv_status p2p_push_chunks(const tsv_verify_args* a, int32_t G, int32_t* chunk, int32_t* NC, int32_t* n_chunks) {
    const int64_t v_max = ((static_cast<int64_t>(a->vocab_global) + G - 1) / G + 3) / 4 * 4;
    int64_t c;
    if (a->chunk > 0) {
        c = a->chunk;
    } else {
        const int64_t warps = static_cast<int64_t>(sm_count()) * 32;
        const int64_t per_row = std::max<int64_t>(1, warps / std::max<int32_t>(a->B, 1));
        c = (v_max + per_row - 1) / per_row;
        c = std::max<int64_t>(512, (c + 127) / 128 * 128);
    }
    if ((v_max + c - 1) / c > kP2PMaxChunks) c = ((v_max + kP2PMaxChunks - 1) / kP2PMaxChunks + 127) / 128 * 128;
    TSV_REQUIRE(c <= kMaxChunk, "tsv_verify p2p fused: chunk %lld > %d", (long long)c, kMaxChunk);
    const int64_t nc = (v_max + c - 1) / c, mine = (static_cast<int64_t>(a->vocab) + c - 1) / c;
    TSV_REQUIRE(nc <= kP2PMaxChunks, "tsv_verify p2p fused: %lld chunks per row > %d (use a larger chunk)",
                (long long)nc, kP2PMaxChunks);
    TSV_REQUIRE(mine <= nc, "tsv_verify p2p fused: shard of %d columns needs %lld chunks of %lld > NC = %lld "
                "(shards up to about ceil4(vocab_global / world) = %lld columns)", a->vocab, (long long)mine,
                (long long)c, (long long)nc, (long long)v_max);
    *chunk = static_cast<int32_t>(c);
    *NC = static_cast<int32_t>(nc);
    *n_chunks = static_cast<int32_t>(mine);
    return TSV_OK;
}

static tsv_status validate(const tsv_verify_args* a) {
    TSV_REQUIRE(a != nullptr, "tsv_verify: args is NULL");
    TSV_REQUIRE(a->B >= 0, "tsv_verify: B < 0 (%d)", a->B);
    TSV_REQUIRE(a->k_max >= 0 && a->k_max <= TSV_MAX_K, "tsv_verify: k_max %d outside [0, %d]", a->k_max, TSV_MAX_K);
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE(a->p && a->row_offsets && a->request_ids && a->num_accepted && a->out_tokens,
                "tsv_verify: a required array is NULL");
    TSV_REQUIRE(a->draft_tokens || a->rows_p == a->B, "tsv_verify: draft_tokens is NULL");
    TSV_REQUIRE(a->ld > 0 && a->ld % 4 == 0, "tsv_verify: ld %lld must be a positive multiple of 4", (long long)a->ld);
    TSV_REQUIRE(aligned16(a->p) && (a->q == nullptr || aligned16(a->q)), "tsv_verify: p/q must be 16-byte aligned");
    TSV_REQUIRE(a->vocab >= 1 && a->vocab <= a->ld, "tsv_verify: vocab %d outside [1, ld]", a->vocab);
    TSV_REQUIRE(a->vocab_offset >= 0 && a->vocab_offset % 4 == 0, "tsv_verify: vocab_offset must be a non-negative multiple of 4");
    TSV_REQUIRE(a->vocab_global >= a->vocab_offset + a->vocab, "tsv_verify: vocab_global < vocab_offset + vocab");
    TSV_REQUIRE(a->rows_p >= a->B, "tsv_verify: rows_p %d < B %d", a->rows_p, a->B);
    TSV_REQUIRE(a->chunk == 0 || (a->chunk >= 128 && a->chunk % 128 == 0 && a->chunk <= kMaxChunk),
                "tsv_verify: chunk must be 0 or a multiple of 128 in [128, %d]", kMaxChunk);
    return TSV_OK;
}

static size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// workspace: [ReqMeta B][rowT rows][rowkey rows] (rows: max(B, rows_p))
static size_t workspace_bytes(const tsv_verify_args* a) {
    const size_t rows = static_cast<size_t>(a->rows_p > a->B ? a->rows_p : a->B);
    return 256 + align256(sizeof(ReqMeta) * static_cast<size_t>(a->B)) + align256(sizeof(uint32_t) * rows) +
           align256(sizeof(uint64_t) * rows);
}

static RaceParams make_params(const tsv_verify_args* a) {
    RaceParams P;
    const int32_t chunk = auto_chunk(a);
    P.p = a->p;
    P.q = a->q;
    P.row_offsets = a->row_offsets;
    P.drafts = a->draft_tokens;
    P.rids = a->request_ids;
    P.num_accepted = a->num_accepted;
    P.out_tokens = a->out_tokens;
    P.devstatus = a->device_status;
    P.step_counts = reinterpret_cast<long long*>(a->step_counts);
    P.tuples = nullptr;
    P.lstats = nullptr;
    P.inv_tau = 1.0f;
    P.ld = a->ld;
    P.k0 = static_cast<uint32_t>(a->seed & 0xFFFFFFFFull);
    P.k1 = static_cast<uint32_t>(a->seed >> 32);
    for (uint32_t r = 0; r < 10; ++r) {
        P.ks0[r] = P.k0 + r * kPhiloxW0;
        P.ks1[r] = P.k1 + r * kPhiloxW1;
    }
    P.step = a->step;
    P.B = a->B;
    P.k_max = a->k_max;
    P.vocab = a->vocab;
    P.vocab_offset = a->vocab_offset;
    P.vocab_global = a->vocab_global;
    P.chunk = chunk;
    P.n_chunks = (a->vocab + chunk - 1) / chunk;
    P.race_update = 0;
    P.ua = UpdateArgs{};
    P.push = 0;
    P.pv = P2PView{};
    P.meta_ready = (a->flags & TSV_VERIFY_META_READY) ? 1 : 0;
    P.early_trigger = (a->flags & TSV_VERIFY_EARLY_TRIGGER) ? 1 : 0;
    P.alpha_ready = nullptr;
    P.rows_p = a->rows_p;
    const size_t n_chunks = static_cast<size_t>(P.n_chunks);
    const size_t rows = static_cast<size_t>(a->rows_p > a->B ? a->rows_p : a->B);
    (void)n_chunks;
    char* ws = static_cast<char*>(a->workspace);
    ws += 256;  // reserved header
    P.meta = reinterpret_cast<ReqMeta*>(ws);
    ws += align256(sizeof(ReqMeta) * static_cast<size_t>(a->B));
    P.rowT = reinterpret_cast<uint32_t*>(ws);
    ws += align256(sizeof(uint32_t) * rows);
    P.rowkey = reinterpret_cast<unsigned long long*>(ws);
    return P;
}

static int sm_count() {
    static int n[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!n[dev]) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
    return n[dev] > 0 ? n[dev] : 148;
}

template <int MODE, bool DENSE_Q, bool PRUNE, bool LOGITS = false, bool PUSH = false>
static tsv_status launch_race(const RaceParams& P, cudaStream_t st) {
    auto kern = verify_race_kernel<MODE, DENSE_Q, PRUNE, LOGITS, PUSH>;
    static int occ = 0;  // resident CTAs per SM
    if (!occ) {
        int b = 0;
        TSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kRaceThreads, 0), "occupancy");
        occ = b > 0 ? b : 1;
    }
    const int64_t per_req = (MODE == kLazy) ? P.n_chunks : static_cast<int64_t>(P.k_max + 1) * P.n_chunks;
    const int64_t n_items = static_cast<int64_t>(P.B) * per_req;
    TSV_REQUIRE(n_items < (1ll << 31), "verify: too many work items");
    const int64_t want = (n_items + kRaceWarps - 1) / kRaceWarps;
    const int64_t base = std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(sm_count()) * occ));
    RaceParams Q = P;
    if (MODE == kLazy && Q.race_update)  // the update on an item-less last warp if there is one, else an extra CTA
        Q.race_update = (TSV_UPDATE_WARP && n_items < base * kRaceWarps) ? 2 : 1;
    const int64_t grid = base + ((MODE == kLazy && Q.race_update == 1) ? 1 : 0);
    TSV_CUDA(launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(kRaceThreads), 0, st, Q), "verify_race_kernel launch");
    return TSV_OK;
}

template <int MODE>
static tsv_status run_verify(const tsv_verify_args* a, RaceParams P, cudaStream_t st, const UpdateArgs* ua = nullptr) {
    const bool race_only = (a->flags & TSV_VERIFY_RACE_ONLY) != 0;  // measurement of the dominant kernel
#ifndef TSV_UPDATE_IN_RACE
#define TSV_UPDATE_IN_RACE 1
#endif
    if (TSV_UPDATE_IN_RACE && MODE == kLazy && ua && !race_only) {  // the alpha update beside the race
        P.race_update = 1;
        P.ua = *ua;
        ua = nullptr;
    }
    const unsigned scan_blocks = static_cast<unsigned>((a->B + 7) / 8);
    if (!race_only)
        TSV_CUDA(launch_pdl(verify_scan_kernel<MODE>, dim3(scan_blocks), dim3(256), 0, st, P), "verify_scan_kernel launch");
    const bool prune = !(a->flags & TSV_VERIFY_NO_PRUNE);
    tsv_status rs;
    if (a->q) rs = prune ? launch_race<MODE, true, true>(P, st) : launch_race<MODE, true, false>(P, st);
    else rs = prune ? launch_race<MODE, false, true>(P, st) : launch_race<MODE, false, false>(P, st);
    TSV_TRY(rs);
    if (race_only) return TSV_OK;
    const unsigned emit_blocks = static_cast<unsigned>((a->B + 7) / 8) + (ua ? 1u : 0u);
    const UpdateArgs none = {};
    cudaError_t e;
    if (ua) e = prune ? launch_pdl(verify_emit_kernel<MODE, true, true>, dim3(emit_blocks), dim3(256), 0, st, P, *ua)
                      : launch_pdl(verify_emit_kernel<MODE, false, true>, dim3(emit_blocks), dim3(256), 0, st, P, *ua);
    else e = prune ? launch_pdl(verify_emit_kernel<MODE, true, false>, dim3(emit_blocks), dim3(256), 0, st, P, none)
                   : launch_pdl(verify_emit_kernel<MODE, false, false>, dim3(emit_blocks), dim3(256), 0, st, P, none);
    TSV_CUDA(e, "verify_emit_kernel launch");
    return TSV_OK;
}

#if TSV_COUNT_EXACT
extern "C" TSV_API void tsv_debug_exact_count(unsigned long long* out) {  // diagnostic builds only
    cudaMemcpyFromSymbol(out, g_exact_count, sizeof(g_exact_count));
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_exact_count, z, sizeof(z));
}
#endif
}  // namespace tsv

using namespace tsv;
TSV_STEP_TRACE_READER(verify)

extern "C" tsv_status tsv_verify_workspace_size(const tsv_verify_args* a, size_t* bytes) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(bytes != nullptr, "tsv_verify_workspace_size: bytes is NULL");
    TSV_TRY(validate(a));
    *bytes = workspace_bytes(a);
    return TSV_OK;
}

extern "C" tsv_status tsv_workspace_clear(void* workspace, size_t bytes, void* stream) {
    TSV_TRACE_CALL();
    if (bytes == 0) return TSV_OK;
    TSV_REQUIRE(workspace != nullptr, "tsv_workspace_clear: workspace is NULL");
    TSV_CUDA(cudaMemsetAsync(workspace, 0, bytes, static_cast<cudaStream_t>(stream)), "cudaMemsetAsync");
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_accept(const tsv_verify_args* a, void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    TSV_REQUIRE(a->vocab_offset == 0 && a->vocab == a->vocab_global,
                "tsv_verify_accept: unsharded call needs vocab_offset == 0 and vocab == vocab_global "
                "(use tsv_verify_shard_partial/combine for vocab shards)");
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE_WS(a->workspace != nullptr && a->workspace_bytes >= workspace_bytes(a),
                "tsv_verify_accept: workspace too small (%llu < %llu bytes)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)workspace_bytes(a));
    TSV_TRY(check_device());
    return run_verify<kLazy>(a, make_params(a), static_cast<cudaStream_t>(stream));
}

extern "C" tsv_status tsv_verify_accept_update(const tsv_verify_args* a, double* alpha, int32_t per_request,
                                               double decay, int32_t estimator, void* stream) {
    TSV_TRACE_CALL();
    return tsv_verify_accept_update_ex(a, alpha, per_request, decay, estimator, nullptr, stream);
}

extern "C" tsv_status tsv_verify_accept_update_ex(const tsv_verify_args* a, double* alpha, int32_t per_request,
                                                  double decay, int32_t estimator, uint32_t* alpha_ready,
                                                  void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    TSV_REQUIRE(a->vocab_offset == 0 && a->vocab == a->vocab_global,
                "tsv_verify_accept_update: unsharded call needs vocab_offset == 0 and vocab == vocab_global");
    TSV_REQUIRE(alpha != nullptr, "tsv_verify_accept_update: alpha is NULL");
    TSV_REQUIRE(decay >= 0.0 && decay <= 1.0, "tsv_verify_accept_update: decay %g outside [0, 1]", decay);
    TSV_REQUIRE(estimator == TSV_EST_TESTED || estimator == TSV_EST_PROPOSED, "tsv_verify_accept_update: unknown estimator");
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE_WS(a->workspace != nullptr && a->workspace_bytes >= workspace_bytes(a),
                "tsv_verify_accept_update: workspace too small (%llu < %llu bytes)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)workspace_bytes(a));
    TSV_TRY(check_device());
    UpdateArgs ua = {};
    ua.alpha = alpha;
    ua.num_accepted = a->num_accepted;
    ua.row_offsets = a->row_offsets;
    ua.decay = decay;
    ua.per_request = per_request;
    ua.B = a->B;
    ua.estimator = estimator;
    ua.alpha_ready = alpha_ready;
    RaceParams P = make_params(a);
    P.alpha_ready = alpha_ready;
    return run_verify<kLazy>(a, P, static_cast<cudaStream_t>(stream), &ua);
}

extern "C" tsv_status tsv_verify_accept_update_p2p(const tsv_verify_args* a, double* alpha, int32_t per_request,
                                                   double decay, int32_t estimator, tsv_p2p* p, void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    TSV_REQUIRE(a->vocab_offset == 0 && a->vocab == a->vocab_global,
                "tsv_verify_accept_update_p2p: needs the whole vocabulary (request-sharded mode)");
    TSV_REQUIRE(alpha != nullptr && p != nullptr, "tsv_verify_accept_update_p2p: NULL argument");
    TSV_REQUIRE(decay >= 0.0 && decay <= 1.0, "tsv_verify_accept_update_p2p: decay %g outside [0, 1]", decay);
    TSV_REQUIRE(estimator == TSV_EST_TESTED || estimator == TSV_EST_PROPOSED,
                "tsv_verify_accept_update_p2p: unknown estimator");
    if (a->B == 0)  // no local requests: this rank still takes part in the exchange (zero sums)
        return tsv_update_acceptance_p2p(alpha, per_request, a->num_accepted, a->row_offsets, 0, decay, estimator, p,
                                         a->device_status, stream);
    TSV_REQUIRE_WS(a->workspace != nullptr && a->workspace_bytes >= workspace_bytes(a),
                   "tsv_verify_accept_update_p2p: workspace too small (%llu < %llu bytes)",
                   (unsigned long long)a->workspace_bytes, (unsigned long long)workspace_bytes(a));
    TSV_TRY(check_device());
    UpdateArgs ua = {};
    ua.alpha = alpha;
    ua.num_accepted = a->num_accepted;
    ua.row_offsets = a->row_offsets;
    ua.decay = decay;
    ua.per_request = per_request;
    ua.B = a->B;
    ua.estimator = estimator;
    ua.use_p2p = per_request ? 0 : 1;
    ua.devstatus = a->device_status;
    ua.p2p = p->view;
    return run_verify<kLazy>(a, make_params(a), static_cast<cudaStream_t>(stream), &ua);
}

extern "C" tsv_status tsv_verify_shard_partial(const tsv_verify_args* a, tsv_shard_tuple* tuples_out,
                                               void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE_WS(a->workspace != nullptr && a->workspace_bytes >= workspace_bytes(a),
                "tsv_verify_shard_partial: workspace too small (%llu < %llu bytes)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)workspace_bytes(a));
    TSV_REQUIRE(tuples_out != nullptr, "tsv_verify_shard_partial: tuples_out is NULL");
    TSV_TRY(check_device());
    RaceParams P = make_params(a);
    P.tuples = tuples_out;
    return run_verify<kShard>(a, P, static_cast<cudaStream_t>(stream));
}

extern "C" tsv_status tsv_verify_shard_combine(const tsv_verify_args* a, const tsv_shard_tuple* gathered,
                                               int32_t num_shards, void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    if (a->B == 0) return TSV_OK;
    TSV_TRY(check_device());
    TSV_REQUIRE(gathered != nullptr, "tsv_verify_shard_combine: gathered is NULL");
    TSV_REQUIRE(num_shards >= 1, "tsv_verify_shard_combine: num_shards < 1");
    RaceParams P = make_params(a);
    const int threads = 256;
    const int64_t blocks = (static_cast<int64_t>(a->B) + (threads / 32) - 1) / (threads / 32);
    TSV_CUDA(launch_pdl(verify_shard_combine_kernel, dim3(static_cast<unsigned>(blocks)), dim3(threads), 0,
                        static_cast<cudaStream_t>(stream), P, gathered, num_shards, a->rows_p),
             "verify_shard_combine_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_shard_flags(const tsv_verify_args* a, uint64_t* masks_out, void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    if (a->B == 0) return TSV_OK;
    TSV_TRY(check_device());
    TSV_REQUIRE(masks_out != nullptr, "tsv_verify_shard_flags: masks_out is NULL");
    RaceParams P = make_params(a);
    TSV_CUDA(launch_pdl(verify_shard_flags_kernel, dim3(static_cast<unsigned>((a->B + 7) / 8)), dim3(256), 0,
                        static_cast<cudaStream_t>(stream), P, reinterpret_cast<unsigned long long*>(masks_out)),
             "verify_shard_flags_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_shard_race(const tsv_verify_args* a, const uint64_t* masks, uint64_t* keys_out,
                                            void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE_WS(a->workspace != nullptr && a->workspace_bytes >= workspace_bytes(a),
                "tsv_verify_shard_race: workspace too small (%llu < %llu bytes)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)workspace_bytes(a));
    TSV_REQUIRE(masks && keys_out, "tsv_verify_shard_race: NULL argument");
    TSV_TRY(check_device());
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    RaceParams P = make_params(a);
    const dim3 grid(static_cast<unsigned>((a->B + 7) / 8));
    TSV_CUDA(launch_pdl(verify_shard_meta_kernel, grid, dim3(256), 0, st, P,
                        reinterpret_cast<const unsigned long long*>(masks)),
             "verify_shard_meta_kernel launch");
    const bool prune = !(a->flags & TSV_VERIFY_NO_PRUNE);
    tsv_status rs;
    if (a->q) rs = prune ? launch_race<kLazy, true, true>(P, st) : launch_race<kLazy, true, false>(P, st);
    else rs = prune ? launch_race<kLazy, false, true>(P, st) : launch_race<kLazy, false, false>(P, st);
    TSV_TRY(rs);
    auto* k = reinterpret_cast<unsigned long long*>(keys_out);
    TSV_CUDA(prune ? launch_pdl(verify_shard_keys_kernel<true>, grid, dim3(256), 0, st, P, k)
                   : launch_pdl(verify_shard_keys_kernel<false>, grid, dim3(256), 0, st, P, k),
             "verify_shard_keys_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_shard_emit(const tsv_verify_args* a, const uint64_t* masks, const uint64_t* keys,
                                            void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    if (a->B == 0) return TSV_OK;
    TSV_TRY(check_device());
    TSV_REQUIRE(masks && keys, "tsv_verify_shard_emit: NULL argument");
    RaceParams P = make_params(a);
    TSV_CUDA(launch_pdl(verify_shard_emit_kernel, dim3(static_cast<unsigned>((a->B + 7) / 8)), dim3(256), 0,
                        static_cast<cudaStream_t>(stream), P, reinterpret_cast<const unsigned long long*>(masks),
                        reinterpret_cast<const unsigned long long*>(keys)),
             "verify_shard_emit_kernel launch");
    return TSV_OK;
}

#if TSV_TRACE
extern "C" TSV_API tsv_status tsv_debug_trace(unsigned long long* out, int32_t n) {
    TSV_TRACE_CALL();
    TSV_CUDA(cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * 4 * static_cast<size_t>(n)), "trace copy");
    return TSV_OK;
}
extern "C" TSV_API tsv_status tsv_debug_trace_clear() {
    TSV_TRACE_CALL();
    static unsigned long long zeros[kTraceMax][4];
    TSV_CUDA(cudaMemcpyToSymbol(g_trace, zeros, sizeof(zeros)), "trace clear");
    return TSV_OK;
}
#endif

extern "C" tsv_status tsv_verify_greedy(const tsv_verify_args* a, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(a != nullptr, "tsv_verify_greedy: args is NULL");
    TSV_REQUIRE(a->B >= 0, "tsv_verify_greedy: B < 0 (%d)", a->B);
    TSV_REQUIRE(a->k_max >= 0 && a->k_max <= TSV_MAX_K, "tsv_verify_greedy: k_max %d outside [0, %d]", a->k_max, TSV_MAX_K);
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE(a->p && a->row_offsets && a->num_accepted && a->out_tokens, "tsv_verify_greedy: a required array is NULL");
    TSV_REQUIRE(a->draft_tokens || a->rows_p == a->B, "tsv_verify_greedy: draft_tokens is NULL");
    TSV_REQUIRE(a->ld > 0 && a->ld % 4 == 0, "tsv_verify_greedy: ld %lld must be a positive multiple of 4", (long long)a->ld);
    TSV_REQUIRE(aligned16(a->p), "tsv_verify_greedy: p must be 16-byte aligned");
    TSV_REQUIRE(a->vocab >= 1 && a->vocab <= a->ld, "tsv_verify_greedy: vocab %d outside [1, ld]", a->vocab);
    TSV_REQUIRE(a->vocab_offset == 0, "tsv_verify_greedy: vocab sharding is not supported");
    TSV_REQUIRE(a->rows_p >= a->B, "tsv_verify_greedy: rows_p %d < B %d", a->rows_p, a->B);
    TSV_REQUIRE(a->chunk == 0 || (a->chunk >= 128 && a->chunk % 128 == 0 && a->chunk <= kMaxChunk),
                "tsv_verify_greedy: chunk must be 0 or a multiple of 128 in [128, %d]", kMaxChunk);
    TSV_REQUIRE_WS(a->workspace != nullptr && a->workspace_bytes >= workspace_bytes(a),
                "tsv_verify_greedy: workspace too small (%llu < %llu bytes)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)workspace_bytes(a));
    TSV_TRY(check_device());
    tsv_verify_args b = *a;
#ifndef TSV_GREEDY_ITEM_WARPS  // items per SM: two per resident warp (config 2: 30.4 us; one: 32.1; 1/2: 32.3)
#define TSV_GREEDY_ITEM_WARPS (2 * 8 * TSV_GREEDY_MINB)
#endif
    if (b.chunk == 0) {  // about two items per resident warp of the argmax grid over all rows
        const int64_t warps = static_cast<int64_t>(sm_count()) * TSV_GREEDY_ITEM_WARPS;
        int64_t c = (static_cast<int64_t>(a->rows_p) * a->vocab + warps - 1) / warps;
        c = (c + 127) / 128 * 128;
        b.chunk = static_cast<int32_t>(std::min<int64_t>(std::max<int64_t>(c, 1024), kMaxChunk));
    }
    RaceParams P = make_params(&b);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
#ifndef TSV_GREEDY_CLEAR_KERNEL
#define TSV_GREEDY_CLEAR_KERNEL 1
#endif
    if (TSV_GREEDY_CLEAR_KERNEL)  // a PDL kernel (its launch overlaps the previous kernel; a memset node does not)
        TSV_CUDA(launch_pdl(clear_u64_kernel, dim3(static_cast<unsigned>((a->rows_p + 1023) / 1024)), dim3(256), 0, st,
                            P.rowkey, static_cast<int64_t>(a->rows_p), P.step_counts),
                 "clear_u64_kernel launch");
    else {
        TSV_CUDA(cudaMemsetAsync(P.rowkey, 0, sizeof(unsigned long long) * static_cast<size_t>(a->rows_p), st),
                 "cudaMemsetAsync");
        if (P.step_counts) TSV_CUDA(cudaMemsetAsync(P.step_counts, 0, 2 * sizeof(long long), st), "cudaMemsetAsync");
    }
    const int64_t n_items = static_cast<int64_t>(a->rows_p) * P.n_chunks;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((n_items + 7) / 8, static_cast<int64_t>(sm_count()) * TSV_GREEDY_MINB));
    TSV_CUDA(launch_pdl(verify_greedy_argmax_kernel, dim3(static_cast<unsigned>(grid)), dim3(256), 0, st, P),
             "verify_greedy_argmax_kernel launch");
    TSV_CUDA(launch_pdl(verify_greedy_emit_kernel, dim3(static_cast<unsigned>((a->B + 7) / 8)), dim3(256), 0, st, P),
             "verify_greedy_emit_kernel launch");
    return TSV_OK;
}

// Logits workspace: [verify workspace][partials (rows_p + rows_p) x n_chunks][lstats B]
// The statistics pass streams every p and q row: its items are sized for ~one per resident warp
// of ITS grid over all rows (so a row has only a few partials for the scan to combine), not the
// lazy race's one-row-per-request items.  An explicit chunk is used for both passes (tests).
#ifndef TSV_STATS_OWN_CHUNK
#define TSV_STATS_OWN_CHUNK 1
#endif
static RaceParams stats_params(const tsv_verify_args* a, RaceParams P) {
    if (a->chunk > 0 || !TSV_STATS_OWN_CHUNK) return P;
#ifndef TSV_STATS_ITEMS_PER_WARP
#define TSV_STATS_ITEMS_PER_WARP 2
#endif
    const int64_t warps = static_cast<int64_t>(sm_count()) * 8 * TSV_STATS_MINB * TSV_STATS_ITEMS_PER_WARP;
    const int64_t cells = 2 * static_cast<int64_t>(a->rows_p) * a->vocab;  // >= (rows_p + rows_q) V
    int64_t c = (cells + warps - 1) / warps;
    c = (c + 127) / 128 * 128;
    if (c < 512) c = 512;
    if (c > (1 << 20)) c = 1 << 20;
    P.chunk = static_cast<int32_t>(c);
    P.n_chunks = static_cast<int32_t>((a->vocab + c - 1) / c);
    return P;
}

static size_t logits_extra_bytes(const tsv_verify_args* a, int32_t n_chunks) {
    return align256(sizeof(LogitPartial) * 2 * static_cast<size_t>(a->rows_p) * static_cast<size_t>(n_chunks)) +
           align256(sizeof(float4) * static_cast<size_t>(a->B));
}

extern "C" tsv_status tsv_verify_logits_workspace_size(const tsv_verify_args* a, size_t* bytes) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(bytes != nullptr, "tsv_verify_logits_workspace_size: bytes is NULL");
    TSV_TRY(validate(a));
    const RaceParams P = stats_params(a, make_params(a));
    *bytes = align256(workspace_bytes(a)) + logits_extra_bytes(a, P.n_chunks);
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_accept_logits(const tsv_verify_args* a, float temperature, void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    TSV_REQUIRE(a->vocab_offset == 0 && a->vocab == a->vocab_global,
                "tsv_verify_accept_logits: vocab sharding is not supported");
    TSV_REQUIRE(temperature > 0.0f && temperature < INFINITY, "tsv_verify_accept_logits: temperature %g must be > 0",
                static_cast<double>(temperature));
    if (a->B == 0) return TSV_OK;
    TSV_TRY(check_device());
    RaceParams P = make_params(a);
    RaceParams PS = stats_params(a, P);  // statistics pass + scan (partials per row)
    const size_t need = align256(workspace_bytes(a)) + logits_extra_bytes(a, PS.n_chunks);
    TSV_REQUIRE_WS(a->workspace != nullptr && a->workspace_bytes >= need,
                "tsv_verify_accept_logits: workspace too small (%llu < %llu bytes)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)need);
    char* ws = static_cast<char*>(a->workspace) + align256(workspace_bytes(a));
    LogitPartial* part = reinterpret_cast<LogitPartial*>(ws);
    ws += align256(sizeof(LogitPartial) * 2 * static_cast<size_t>(a->rows_p) * static_cast<size_t>(PS.n_chunks));
    float4* lstats = reinterpret_cast<float4*>(ws);
    P.lstats = PS.lstats = lstats;
    P.inv_tau = PS.inv_tau = static_cast<float>(1.0 / static_cast<double>(temperature));
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n_items = 2 * static_cast<int64_t>(a->rows_p) * PS.n_chunks;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((n_items + 7) / 8, static_cast<int64_t>(sm_count()) * TSV_STATS_MINB));
    TSV_CUDA(launch_pdl(verify_logit_stats_kernel, dim3(static_cast<unsigned>(grid)), dim3(256), 0, st, PS, part,
                        a->rows_p - a->B),
             "verify_logit_stats_kernel launch");
    const dim3 req_grid(static_cast<unsigned>((a->B + 7) / 8));
    TSV_CUDA(launch_pdl(verify_logit_scan_kernel, req_grid, dim3(256), 0, st, PS,
                        static_cast<const LogitPartial*>(part), lstats),
             "verify_logit_scan_kernel launch");
    const bool prune = !(a->flags & TSV_VERIFY_NO_PRUNE);
    tsv_status rs;
    if (a->q) rs = prune ? launch_race<kLazy, true, true, true>(P, st) : launch_race<kLazy, true, false, true>(P, st);
    else rs = prune ? launch_race<kLazy, false, true, true>(P, st) : launch_race<kLazy, false, false, true>(P, st);
    TSV_TRY(rs);
    const UpdateArgs none = {};
    TSV_CUDA(prune ? launch_pdl(verify_emit_kernel<kLazy, true, false, true>, req_grid, dim3(256), 0, st, P, none)
                   : launch_pdl(verify_emit_kernel<kLazy, false, false, true>, req_grid, dim3(256), 0, st, P, none),
             "verify_emit_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_softmax_rows(const float* z, int64_t ld, int32_t vocab, int32_t rows, float temperature,
                                       float* p_out, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(rows >= 0, "tsv_softmax_rows: rows < 0");
    TSV_REQUIRE(vocab >= 1 && vocab <= ld, "tsv_softmax_rows: vocab %d outside [1, ld]", vocab);
    TSV_REQUIRE(temperature > 0.0f && temperature < INFINITY, "tsv_softmax_rows: temperature must be > 0");
    if (rows == 0) return TSV_OK;
    TSV_REQUIRE(z && p_out, "tsv_softmax_rows: NULL argument");
    TSV_TRY(check_device());
    const float inv_tau = static_cast<float>(1.0 / static_cast<double>(temperature));
    TSV_CUDA(launch_pdl(softmax_rows_kernel, dim3(static_cast<unsigned>(rows)), dim3(256), 0,
                        static_cast<cudaStream_t>(stream), z, ld, vocab, inv_tau, p_out),
             "softmax_rows_kernel launch");
    return TSV_OK;
}

// ------------------------------------------------------------------ diagnostics (tests)
namespace tsv {
// One warp races one row of weights with INJECTED Philox words (instead of generated ones),
// through exactly the race kernel's Race logic: prune test, deferred exact evaluation, packed
// keys.  Lets the GPU tests drive adversarial words (identical words -> exact score ties).
template <bool PRUNE>
__global__ void debug_race_row_kernel(const float* __restrict__ w, const uint32_t* __restrict__ words, int32_t V,
                                      unsigned long long* key_out) {
    const int lane = threadIdx.x & 31;
    const int32_t nq = (V + 3) >> 2;
    Race R;
    R.init();
    for (int32_t f0 = 0; f0 < nq; f0 += 32) {
        const int32_t f = f0 + lane;
        float wv[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t x[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int32_t v = 4 * f + t;
            if (f < nq && v < V) {
                wv[t] = w[v];
                x[t] = words[v];
            }
        }
        const uint4 r = make_uint4(x[0], x[1], x[2], x[3]);
        if (PRUNE && R.T == 0.0f) R.warm(wv, r);
        R.quad<PRUNE>(wv, r, static_cast<uint32_t>(4 * f));
        if (PRUNE) R.sync_T();
    }
    R.finish<PRUNE>(R.T);
    const uint64_t key = warp_max_u64(R.best);
    if (lane == 0) *key_out = key;
}
}  // namespace tsv

extern "C" tsv_status tsv_debug_race_row(const float* w, const uint32_t* words, int32_t V, int32_t prune,
                                         uint64_t* key_out, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(w && words && key_out && V >= 1, "tsv_debug_race_row: bad arguments");
    TSV_TRY(check_device());
    auto* k = reinterpret_cast<unsigned long long*>(key_out);
    if (prune) debug_race_row_kernel<true><<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(w, words, V, k);
    else debug_race_row_kernel<false><<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(w, words, V, k);
    TSV_CUDA(cudaGetLastError(), "debug_race_row_kernel launch");
    return TSV_OK;
}

// ------------------------------------------------------------ peer-memory vocab sharding (host)

extern "C" tsv_status tsv_p2p_buffer_size(int32_t B_max, size_t* bytes) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(bytes != nullptr && B_max >= 1, "tsv_p2p_buffer_size: bad arguments");
    *bytes = tsv::p2p_buffer_bytes(B_max);
    return TSV_OK;
}

extern "C" tsv_status tsv_p2p_alloc(int32_t B_max, void** buf_out, void* ipc_handle_out) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(buf_out != nullptr && B_max >= 1, "tsv_p2p_alloc: bad arguments");
    TSV_TRY(check_device());
    void* p = nullptr;
    const size_t n = tsv::p2p_buffer_bytes(B_max);
    TSV_CUDA(cudaMalloc(&p, n), "cudaMalloc (p2p buffer)");
    TSV_CUDA(cudaMemset(p, 0, n), "cudaMemset (p2p buffer)");
    if (ipc_handle_out) {
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        cudaIpcMemHandle_t h;
        TSV_CUDA(cudaIpcGetMemHandle(&h, p), "cudaIpcGetMemHandle");
        memcpy(ipc_handle_out, &h, sizeof(h));
    }
    *buf_out = p;
    return TSV_OK;
}

extern "C" tsv_status tsv_p2p_free(void* buf) {
    TSV_TRACE_CALL();
    if (buf) TSV_CUDA(cudaFree(buf), "cudaFree (p2p buffer)");
    return TSV_OK;
}

extern "C" tsv_status tsv_p2p_open(const void* ipc_handle, void** buf_out) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(ipc_handle && buf_out, "tsv_p2p_open: NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    TSV_CUDA(cudaIpcOpenMemHandle(buf_out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    return TSV_OK;
}

extern "C" tsv_status tsv_p2p_close(void* buf) {
    TSV_TRACE_CALL();
    if (buf) TSV_CUDA(cudaIpcCloseMemHandle(buf), "cudaIpcCloseMemHandle");
    return TSV_OK;
}

extern "C" tsv_status tsv_p2p_init(tsv_p2p** out, int32_t rank, int32_t world, int32_t B_max, void* const* bufs) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(out && bufs, "tsv_p2p_init: NULL argument");
    TSV_REQUIRE(world >= 1 && world <= TSV_P2P_MAX_WORLD && rank >= 0 && rank < world && B_max >= 1,
                "tsv_p2p_init: rank %d / world %d / B_max %d invalid", rank, world, B_max);
    auto* p = new tsv_p2p;
    memset(&p->view, 0, sizeof(p->view));
    for (int32_t g = 0; g < world; ++g) {
        TSV_REQUIRE(bufs[g] != nullptr, "tsv_p2p_init: buffer of rank %d is NULL", g);
        p->view.buf[g] = static_cast<unsigned char*>(bufs[g]);
    }
    p->view.rank = rank;
    p->view.G = world;
    p->view.B_max = B_max;
    *out = p;
    return TSV_OK;
}

extern "C" tsv_status tsv_p2p_destroy(tsv_p2p* p) {
    TSV_TRACE_CALL();
    delete p;
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_shard_p2p_phase(const tsv_verify_args* a, tsv_p2p* p, int32_t phase, void* stream) {
    TSV_TRACE_CALL();
    TSV_TRY(validate(a));
    TSV_REQUIRE(p != nullptr, "tsv_verify_shard_p2p_phase: p2p handle is NULL");
    TSV_REQUIRE(phase >= 0 && phase <= 2, "tsv_verify_shard_p2p_phase: phase %d", phase);
    TSV_REQUIRE(a->B <= p->view.B_max, "tsv_verify_shard_p2p_phase: B %d > B_max %d", a->B, p->view.B_max);
    TSV_REQUIRE_WS(a->workspace != nullptr && a->workspace_bytes >= workspace_bytes(a),
                "tsv_verify_shard_p2p_phase: workspace too small (%llu < %llu bytes)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)workspace_bytes(a));
    TSV_TRY(check_device());
    if (a->B == 0) return TSV_OK;  // (all ranks skip the exchange together; the epoch does not advance)
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    RaceParams P = make_params(a);
    const dim3 grid(static_cast<unsigned>((a->B + 7) / 8));
    const P2PView V = p->view;
    const bool prune = !(a->flags & TSV_VERIFY_NO_PRUNE);
    const bool fused = (a->flags & TSV_VERIFY_P2P_FUSED) != 0;
    int32_t NC = 0;  // fused: chunks per row polled per rank, identical on every rank
    if (fused) TSV_TRY(p2p_push_chunks(a, V.G, &P.chunk, &NC, &P.n_chunks));
    if (phase == 0) {
        TSV_CUDA(launch_pdl(verify_p2p_flags_kernel, grid, dim3(256), 0, st, P, V, NC), "verify_p2p_flags_kernel launch");
    } else if (phase == 1) {
        TSV_CUDA(launch_pdl(verify_p2p_meta_kernel, grid, dim3(256), 0, st, P, V), "verify_p2p_meta_kernel launch");
        tsv_status rs;
        if (fused) {
            P.push = 1;
            P.pv = V;
            if (a->q) rs = prune ? launch_race<kLazy, true, true, false, true>(P, st) : launch_race<kLazy, true, false, false, true>(P, st);
            else rs = prune ? launch_race<kLazy, false, true, false, true>(P, st) : launch_race<kLazy, false, false, false, true>(P, st);
        } else {
            if (a->q) rs = prune ? launch_race<kLazy, true, true>(P, st) : launch_race<kLazy, true, false>(P, st);
            else rs = prune ? launch_race<kLazy, false, true>(P, st) : launch_race<kLazy, false, false>(P, st);
        }
        TSV_TRY(rs);
        if (!fused)
            TSV_CUDA(prune ? launch_pdl(verify_p2p_keys_kernel<true>, grid, dim3(256), 0, st, P, V)
                           : launch_pdl(verify_p2p_keys_kernel<false>, grid, dim3(256), 0, st, P, V),
                     "verify_p2p_keys_kernel launch");
    } else if (fused) {
        TSV_CUDA(prune ? launch_pdl(verify_p2p_emit_push_kernel<true>, grid, dim3(256), 0, st, P, V, NC)
                       : launch_pdl(verify_p2p_emit_push_kernel<false>, grid, dim3(256), 0, st, P, V, NC),
                 "verify_p2p_emit_push_kernel launch");
    } else {
        TSV_CUDA(launch_pdl(verify_p2p_emit_kernel, grid, dim3(256), 0, st, P, V), "verify_p2p_emit_kernel launch");
    }
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_accept_sharded_p2p(const tsv_verify_args* a, tsv_p2p* p, void* stream) {
    TSV_TRACE_CALL();
    for (int32_t ph = 0; ph < 3; ++ph) TSV_TRY(tsv_verify_shard_p2p_phase(a, p, ph, stream));
    return TSV_OK;
}

extern "C" tsv_status tsv_allreduce_i64_p2p(int64_t* data, int32_t count, tsv_p2p* p, int32_t* device_status,
                                           void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(data && p, "tsv_allreduce_i64_p2p: NULL argument");
    TSV_REQUIRE(count >= 0 && count <= TSV_P2P_MAX_SUMS, "tsv_allreduce_i64_p2p: count %d outside [0, %d]", count,
                TSV_P2P_MAX_SUMS);
    TSV_TRY(check_device());
    TSV_CUDA(launch_pdl(p2p_allreduce_i64_kernel, dim3(1), dim3(TSV_P2P_MAX_SUMS), 0, static_cast<cudaStream_t>(stream),
                        data, count, p->view, device_status),
             "p2p_allreduce_i64_kernel launch");
    return TSV_OK;
}
