// verify.cu -- rejection-sampling verify/accept on sm_100a.
// PAPER.md:18 [AD], 493-497 [BG]; readings R1-R9 in DESIGN.md section 3.
//
// One tsv_verify_accept call = three kernels chained with programmatic dependent launch
// (PDL, griddepcontrol), so each kernel's launch and prologue overlap its predecessor:
//
//  1. verify_scan_kernel: one warp per request.  Acceptance test with first-rejection
//     scan (lane j < k_i gathers p_j[x_j], q_j[x_j], draws u_acc, one ballot) -> m_i.
//     Writes a 32-byte ReqMeta per request; bad requests are emitted (-1) right here.
//  2. verify_race_kernel: warp-independent.  Work item = (request, 2048-column chunk) of
//     the selected row [lazy] or (request, position, chunk) of every row [vocab-shard
//     partial], interleaved over all warps of the grid.  Each warp streams its chunk of p
//     -- and of q on a rejection -- with 128-bit loads into registers (2-deep prefetch),
//     one specialised Philox4x32-10 call per float4, the provably conservative prune test
//      that skips the exact double-log + IEEE-division score of elements
//     that cannot reach the best score seen, deferred exact evaluation of survivors, and
//     a packed (score, ~index) u64 key per item, stored without atomics.  No shared
//     memory, no barriers, no inter-warp synchronisation.
//  3. verify_emit_kernel: one warp per request (or p row in shard mode) reduces the
//     chunk keys (max), falls back to the p_m race when the residual was identically zero
//     (R5), and emits out_tokens / num_accepted (or the shard tuple).
#include <stdio.h>

#include <algorithm>

#include "common.cuh"

namespace tsv {

struct ReqMeta {           // 32 bytes, written by the scan kernel
    int32_t r0, k, qbase, m;
    int32_t xm, ok;        // ok: 1 valid, 0 bad k, 2 bad draft token
    uint32_t rid, pad;
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
    ReqMeta* meta;             // [B]
    uint64_t* keys;            // [n_key_rows * n_chunks] race keys
    uint64_t* fbkeys;          // [n_key_rows * n_chunks] fallback keys (valid where key == 0)
    tsv_shard_tuple* tuples;   // shard mode
    int64_t ld;
    uint32_t k0, k1, step;
    int32_t B, k_max, vocab, vocab_offset, vocab_global, chunk, n_chunks, rows_p;
    uint32_t ks0[10], ks1[10];  // Philox key schedule k + r W (constant bank)
};

enum Mode { kLazy = 0, kShard = 1 };

constexpr int kChunk = 2048;                      // columns per work item (default)
constexpr int kMaxChunk = 16384;
constexpr float kPruneC = 0x1.fffffap-1f;        // 1 - 3*2^-24 <= (1-2^-23)(1-2^-24)
constexpr float kLbC = 0x1.ffffe0p-1f;           // 1 - 2^-20
constexpr float kMinNormal = 0x1p-126f;

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Lower bound on the exact score RN32(w / E(u)) of an element:
// E <= (-ln u)(1+2^-24) <= ((1-u)/u)(1+2^-24), and rcp.approx is within 2^-22.
__device__ __forceinline__ float race_lower_bound(float w, float omu) {
    const float u = __fsub_rn(1.0f, omu);  // exact
    return __fmul_rd(__fmul_rd(w, u), __fmul_rd(rcp_approx(omu), kLbC));
}

__device__ __forceinline__ float prune_scale(float T) {
    return T >= kMinNormal ? __fmul_rd(T, kPruneC) : 0.0f;
}

// Per-thread race state.  T is warp-uniform: a lower bound on (or an exact value of) a
// score achieved by an element of this row; Tc = RD(T (1 - 3 2^-24)).
struct Race {
    float T, Tc, Tloc;
    uint64_t best;
    bool has_pend;
    float pend_w, pend_omu;
    uint32_t pend_x, pend_v;

    __device__ __forceinline__ void init() {
        T = Tc = Tloc = 0.0f;
        best = 0;
        has_pend = false;
        pend_w = 0.0f;
        pend_omu = 1.0f;
        pend_x = pend_v = 0;
    }

    __device__ __forceinline__ void eval_exact(float w, uint32_t x, uint32_t vg) {
        const uint64_t key = exact_race_key(w, x, vg);
        best = key > best ? key : best;
        Tloc = fmaxf(Tloc, __uint_as_float(static_cast<uint32_t>(best >> 32)));
    }

    // One float4 of weights w (0 = not a candidate) with Philox words r, global index v0.
    template <bool PRUNE>
    __device__ __forceinline__ void quad(const float (&w)[4], const uint4& r, uint32_t v0) {
        const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
        if constexpr (!PRUNE) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (w[e] > 0.0f) eval_exact(w[e], rw[e], v0 + e);
        } else {
            quad_pruned(w, rw, v0);
        }
    }

    __device__ __forceinline__ void quad_pruned(const float (&w)[4], const uint32_t (&rw)[4], uint32_t v0) {
        float omu[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) omu[e] = one_minus_u_race(rw[e]);
        if (T == 0.0f) {  // warp-uniform warm-up: seed T from lower bounds
            float lb = 0.0f;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (w[e] > 0.0f) lb = fmaxf(lb, race_lower_bound(w[e], omu[e]));
            Tloc = fmaxf(Tloc, lb);
            sync_T();
        }
        bool cand[4];
        bool any = false;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            cand[e] = w[e] > __fmul_rd(Tc, omu[e]);
            any |= cand[e];
        }
        if (any) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (cand[e]) {
                    Tloc = fmaxf(Tloc, race_lower_bound(w[e], omu[e]));
                    if (has_pend && pend_w > __fmul_rd(Tc, pend_omu)) eval_exact(pend_w, pend_x, pend_v);
                    has_pend = true;
                    pend_w = w[e];
                    pend_omu = omu[e];
                    pend_x = rw[e];
                    pend_v = v0 + e;
                }
            }
        }
    }

    __device__ __forceinline__ void sync_T() {  // warp-wide max (REDUX on the float bits)
        T = __uint_as_float(__reduce_max_sync(0xFFFFFFFFu, __float_as_uint(Tloc)));
        Tc = prune_scale(T);
    }

    // Flush the parked candidate against a (possibly CTA-wide) final threshold.
    template <bool PRUNE>
    __device__ __forceinline__ void finish(float T_final) {
        if constexpr (PRUNE) {
            const float tc = prune_scale(T_final);
            if (has_pend && pend_w > __fmul_rd(tc, pend_omu)) eval_exact(pend_w, pend_x, pend_v);
            has_pend = false;
        }
    }
};

// Weights of one float4: residual max(0, p - q) (dense q, or one-hot at local column xm)
// or bonus max(0, p); columns >= col_end are 0.  NaN -> 0 (fmaxf).
template <bool DENSE_Q>
__device__ __forceinline__ void quad_weights(float (&w)[4], const float4& a, const float4& b, bool residual,
                                             int32_t col, int32_t col_end, int32_t xm) {
    const float pv[4] = {a.x, a.y, a.z, a.w};
    const float qv[4] = {b.x, b.y, b.z, b.w};
    if (residual) {
        if (DENSE_Q) {
#pragma unroll
            for (int e = 0; e < 4; ++e) w[e] = fmaxf(__fsub_rn(pv[e], qv[e]), 0.0f);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) w[e] = fmaxf(pv[e], 0.0f);
            if ((col >> 2) == (xm >> 2)) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (col + e == xm) w[e] = fmaxf(__fsub_rn(pv[e], 1.0f), 0.0f);
            }
        }
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) w[e] = fmaxf(pv[e], 0.0f);
    }
    if (col + 4 > col_end) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (col + e >= col_end) w[e] = 0.0f;
    }
}

__device__ __forceinline__ void report(int32_t* devstatus, uint32_t bits) {
    if (devstatus && bits) atomicOr(reinterpret_cast<unsigned int*>(devstatus), bits);
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

// ------------------------------------------------------------------ 1. acceptance scan
// One warp per request (R1-R4).  Lane j < k tests draft j if this shard owns x_j (the
// lazy mode's shard is the whole vocabulary).  Lazy: invalid requests are emitted here.
// Shard: writes the accept / owner flags of every p row of the request into its tuple.
template <int MODE>
__global__ void __launch_bounds__(256) verify_scan_kernel(const RaceParams P) {
    pdl_launch_dependents();  // let the race kernel launch and set up while we scan
    const int32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const int lane = threadIdx.x & 31;
    const int32_t r0 = P.row_offsets[i];
    const int32_t r1 = P.row_offsets[i + 1];
    const int32_t k = r1 - r0 - 1;
    const int32_t qbase = r0 - i;
    int32_t ok = (k >= 0 && k <= P.k_max && qbase >= 0 && r1 <= P.rows_p) ? 1 : 0;
    const uint32_t rid = P.rids[i];
    int32_t x = -1;
    bool bad = false, acc = false, own = false;
    if (ok && lane < k) {
        x = P.drafts[qbase + lane];
        bad = x < 0 || x >= P.vocab_global;
        const int32_t xl = x - P.vocab_offset;
        own = !bad && xl >= 0 && xl < P.vocab;
        if (own) {
            const uint4 rr = philox4x32_10(0u, (kPurposeAccept << 16) | static_cast<uint32_t>(lane), rid, P.step,
                                           P.k0, P.k1);
            const float u = u_acc_from_word(rr.x);
            const float qx = P.q ? P.q[static_cast<int64_t>(qbase + lane) * P.ld + xl] : 1.0f;
            const float px = P.p[static_cast<int64_t>(r0 + lane) * P.ld + xl];
            acc = __fmul_rn(u, qx) < px;  // strict; NaN rejects
        }
    }
    const uint32_t badm = __ballot_sync(0xFFFFFFFFu, bad);
    const uint32_t accm = __ballot_sync(0xFFFFFFFFu, acc);
    const uint32_t ownm = __ballot_sync(0xFFFFFFFFu, own);
    if (badm) ok = 2;
    const uint32_t kmask = (ok == 1 && k > 0) ? ((1u << k) - 1u) : 0u;
    const uint32_t rej = ~accm & kmask;
    const int32_t m = rej ? (__ffs(rej) - 1) : (ok == 1 ? k : -1);
    const int32_t xm = __shfl_sync(0xFFFFFFFFu, x, (m >= 0 ? m : 0) & 31);
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
        if (ok != 1) {
            emit(P, i, 0, -1, -1);
            if (lane == 0) report(P.devstatus, ok == 2 ? TSV_DEVSTATUS_BAD_TOKEN : TSV_DEVSTATUS_BAD_K);
        }
    } else if (ok == 1 && lane <= k) {  // rows j <= k of this request: flags (bit0 accept, bit1 owner)
        const uint32_t flag = lane < k ? (((accm >> lane) & 1u) | (((ownm >> lane) & 1u) << 1)) : 0u;
        P.tuples[r0 + lane].flag = flag;
        P.tuples[r0 + lane].pad = 0;
    }
}

// ------------------------------------------------------------------ 2. the race
// Warp-independent: every warp races its own work items (request [, position], chunk of
// P.chunk columns), statically interleaved over all warps of the grid so residual and
// bonus rows mix on every SM.  Each lane streams float4s of the row chunk straight into
// registers (LDG.128, L1 no-allocate, 256-byte L2 prefetch) with a 2-deep software
// prefetch; no shared memory, no barriers, no atomics.  The item's key is a plain store.
constexpr int kRaceThreads = 256;
constexpr int kRaceWarps = kRaceThreads / 32;

template <int MODE, bool DENSE_Q, bool PRUNE>
__global__ void __launch_bounds__(kRaceThreads, 4) verify_race_kernel(const RaceParams P) {
    pdl_wait();  // the scan kernel's ReqMeta is complete and visible from here on
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t warp_id = static_cast<int64_t>(blockIdx.x) * kRaceWarps + (threadIdx.x >> 5);
    const int64_t n_warps = static_cast<int64_t>(gridDim.x) * kRaceWarps;
    const int32_t per_req = (MODE == kLazy) ? P.n_chunks : (P.k_max + 1) * P.n_chunks;
    const int64_t n_items = static_cast<int64_t>(P.B) * per_req;
    const uint32_t vbase = static_cast<uint32_t>(P.vocab_offset);

    for (int64_t item = warp_id; item < n_items; item += n_warps) {
        const int32_t i = static_cast<int32_t>(item / per_req);
        const int32_t rem = static_cast<int32_t>(item - static_cast<int64_t>(i) * per_req);
        const int32_t j = rem / P.n_chunks;
        const int32_t c = rem - j * P.n_chunks;
        const ReqMeta rm = P.meta[i];
        if (rm.ok != 1) continue;
        const int32_t sel = (MODE == kLazy) ? rm.m : j;
        if (MODE == kShard && sel > rm.k) continue;  // no such row
        const bool residual = sel < rm.k;
        const bool use_q = DENSE_Q && residual;
        int32_t xm_local = -1;
        if (residual && !DENSE_Q) xm_local = ((MODE == kLazy) ? rm.xm : P.drafts[rm.qbase + sel]) - P.vocab_offset;
        const int32_t col_begin = c * P.chunk;
        const int32_t col_end = min(P.vocab, col_begin + P.chunk);
        const float4* prow = reinterpret_cast<const float4*>(P.p + static_cast<int64_t>(rm.r0 + sel) * P.ld + col_begin);
        const float4* qrow = use_q ? reinterpret_cast<const float4*>(P.q + static_cast<int64_t>(rm.qbase + sel) * P.ld + col_begin)
                                   : prow;
        const int32_t nq = (col_end - col_begin + 3) >> 2;
        const int32_t iters = (nq + 31) >> 5;
        const RaceCtr rc = race_ctr((kPurposeRace << 16) | static_cast<uint32_t>(sel), rm.rid, P.step, P.k0, P.k1);

        Race R;
        R.init();
        // full iterations: all 32 lanes in range, two float4 per lane per step, no masking
        const int32_t nfull = (col_end - col_begin) >> 7;  // 32 lanes x 4 columns
        int32_t it = 0;
        for (; it + 1 < nfull; it += 2) {
            const int32_t f0 = it * 32 + lane, f1 = f0 + 32;
            const float4 a0 = ldg_stream(prow + f0);
            const float4 a1 = ldg_stream(prow + f1);
            float4 b0 = make_float4(0.f, 0.f, 0.f, 0.f), b1 = b0;  // read only when use_q
            if (use_q) {
                b0 = ldg_stream(qrow + f0);
                b1 = ldg_stream(qrow + f1);
            }
            const int32_t col0 = col_begin + 4 * f0, col1 = col0 + 128;
            const uint4 r0 = philox_race(rc, (vbase >> 2) + static_cast<uint32_t>(col0 >> 2), P);
            const uint4 r1 = philox_race(rc, (vbase >> 2) + static_cast<uint32_t>(col1 >> 2), P);
            float w0[4], w1[4];
            quad_weights<DENSE_Q>(w0, a0, b0, residual, col0, 0x7FFFFFFF, xm_local);
            quad_weights<DENSE_Q>(w1, a1, b1, residual, col1, 0x7FFFFFFF, xm_local);
            R.quad<PRUNE>(w0, r0, vbase + static_cast<uint32_t>(col0));
            R.quad<PRUNE>(w1, r1, vbase + static_cast<uint32_t>(col1));
            if (PRUNE) R.sync_T();
        }
        // remaining iterations (odd count / ragged tail): bounds checks and column masking
        for (; it < iters; ++it) {
            const int32_t f = it * 32 + lane;
            const int32_t col = col_begin + 4 * f;
            float w[4] = {0.f, 0.f, 0.f, 0.f};
            uint4 r = make_uint4(0, 0, 0, 0);
            if (f < nq) {
                const float4 a = ldg_stream(prow + f);
                const float4 b = use_q ? ldg_stream(qrow + f) : a;
                quad_weights<DENSE_Q>(w, a, b, residual, col, col_end, xm_local);
                r = philox_race(rc, (vbase >> 2) + static_cast<uint32_t>(col >> 2), P);
            }
            R.quad<PRUNE>(w, r, vbase + static_cast<uint32_t>(col));
            if (PRUNE) R.sync_T();
        }
        R.finish<PRUNE>(R.T);
        const uint64_t best = warp_max_u64(R.best);
        uint64_t fb = 0;
        if (best == 0 && residual) {  // residual identically zero on this chunk: race over p (R5)
            Race F;
            F.init();
            for (int32_t it = 0; it < iters; ++it) {
                const int32_t f = it * 32 + lane;
                const int32_t col = col_begin + 4 * f;
                const float4 a = f < nq ? ldg_stream(prow + f) : make_float4(0.f, 0.f, 0.f, 0.f);
                float w[4];
                quad_weights<true>(w, a, a, false, col, col_end, -1);
                const uint4 r = philox_race(rc, (vbase >> 2) + static_cast<uint32_t>(col >> 2), P);
                F.quad<PRUNE>(w, r, vbase + static_cast<uint32_t>(col));
                if (PRUNE) F.sync_T();
            }
            F.finish<PRUNE>(F.T);
            fb = warp_max_u64(F.best);
        }
        if (lane == 0) {
            const int64_t key_index = static_cast<int64_t>(MODE == kLazy ? i : rm.r0 + sel) * P.n_chunks + c;
            P.keys[key_index] = best;
            P.fbkeys[key_index] = fb;
        }
    }
}

// ------------------------------------------------------------------ 3. emit
// Lazy: one warp per request.  Shard: one warp per p row (writes the tuple keys).
template <int MODE>
__global__ void __launch_bounds__(256) verify_emit_kernel(const RaceParams P) {
    pdl_wait();
    const int32_t unit = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (MODE == kLazy) {
        if (unit >= P.B) return;
        const ReqMeta rm = P.meta[unit];
        if (rm.ok != 1) return;  // emitted by the scan kernel
        uint64_t key = 0, fb = 0;
        for (int32_t c = lane; c < P.n_chunks; c += 32) {
            const uint64_t a = P.keys[static_cast<int64_t>(unit) * P.n_chunks + c];
            const uint64_t b = P.fbkeys[static_cast<int64_t>(unit) * P.n_chunks + c];
            key = a > key ? a : key;
            fb = b > fb ? b : fb;
        }
        key = warp_max_u64(key);
        fb = warp_max_u64(fb);
        if (key == 0 && rm.m < rm.k) key = fb;  // R5 (valid: every chunk raced p_m)
        emit(P, unit, rm.qbase, rm.m, key ? key_index(key) : -1);
        if (lane == 0 && !key) report(P.devstatus, TSV_DEVSTATUS_NO_WEIGHT);
    } else {
        if (unit >= P.rows_p) return;
        uint64_t key = 0, fb = 0;
        for (int32_t c = lane; c < P.n_chunks; c += 32) {
            const uint64_t a = P.keys[static_cast<int64_t>(unit) * P.n_chunks + c];
            const uint64_t b = P.fbkeys[static_cast<int64_t>(unit) * P.n_chunks + c];
            key = a > key ? a : key;
            fb = b > fb ? b : fb;
        }
        key = warp_max_u64(key);
        fb = warp_max_u64(fb);
        if (lane == 0) {
            P.tuples[unit].key = key;
            P.tuples[unit].fb_key = key ? 0ull : fb;
        }
    }
}

// ------------------------------------------------------------------------ shard combine
// One warp per request: OR the accept flags of the G shards, scan m, take the max key of
// row m over shards (fallback keys if every shard's residual was zero), emit.
__global__ void verify_shard_combine_kernel(const RaceParams P, const tsv_shard_tuple* __restrict__ g,
                                            int32_t G, int32_t rows_p) {
    const int32_t warps_per_block = blockDim.x >> 5;
    const int32_t i = blockIdx.x * warps_per_block + (threadIdx.x >> 5);
    if (i >= P.B) return;
    const int lane = threadIdx.x & 31;
    const int32_t r0 = P.row_offsets[i];
    const int32_t r1 = P.row_offsets[i + 1];
    const int32_t k = r1 - r0 - 1;
    const int32_t qbase = r0 - i;
    const bool ok = k >= 0 && k <= P.k_max && qbase >= 0 && r1 <= rows_p;
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
        return;
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
}

// ------------------------------------------------------------------------ host side
static int32_t auto_chunk(const tsv_verify_args* a) { return a->chunk > 0 ? a->chunk : kChunk; }

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
    TSV_REQUIRE(a->chunk == 0 || (a->chunk >= 1024 && a->chunk % 1024 == 0 && a->chunk <= kMaxChunk),
                "tsv_verify: chunk must be 0 or a multiple of 1024 in [1024, %d]", kMaxChunk);
    return TSV_OK;
}

static size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// workspace: [ReqMeta B][keys n][fbkeys n], n = key rows * n_chunks (key rows: B lazy, rows_p shard)
static size_t workspace_bytes(const tsv_verify_args* a) {
    const int32_t chunk = auto_chunk(a);
    const size_t n_chunks = static_cast<size_t>((a->vocab + chunk - 1) / chunk);
    const size_t rows = static_cast<size_t>(a->rows_p > a->B ? a->rows_p : a->B);
    return align256(sizeof(ReqMeta) * static_cast<size_t>(a->B)) + 2 * align256(sizeof(uint64_t) * rows * n_chunks);
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
    P.tuples = nullptr;
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
    P.rows_p = a->rows_p;
    const size_t n_chunks = static_cast<size_t>(P.n_chunks);
    const size_t rows = static_cast<size_t>(a->rows_p > a->B ? a->rows_p : a->B);
    char* ws = static_cast<char*>(a->workspace);
    P.meta = reinterpret_cast<ReqMeta*>(ws);
    P.keys = reinterpret_cast<uint64_t*>(ws + align256(sizeof(ReqMeta) * static_cast<size_t>(a->B)));
    P.fbkeys = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(P.keys) + align256(sizeof(uint64_t) * rows * n_chunks));
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

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int MODE, bool DENSE_Q, bool PRUNE>
static tsv_status launch_race(const RaceParams& P, cudaStream_t st) {
    auto kern = verify_race_kernel<MODE, DENSE_Q, PRUNE>;
    static int occ = 0;  // resident CTAs per SM
    if (!occ) {
        int b = 0;
        TSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kRaceThreads, 0), "occupancy");
        occ = b > 0 ? b : 1;
    }
    const int64_t per_req = (MODE == kLazy) ? P.n_chunks : static_cast<int64_t>(P.k_max + 1) * P.n_chunks;
    const int64_t n_items = static_cast<int64_t>(P.B) * per_req;
    const int64_t want = (n_items + kRaceWarps - 1) / kRaceWarps;
    const int64_t grid = std::min<int64_t>(want, static_cast<int64_t>(sm_count()) * occ);
    TSV_CUDA(launch_pdl(kern, dim3(static_cast<unsigned>(grid > 0 ? grid : 1)), dim3(kRaceThreads), 0, st, P),
             "verify_race_kernel launch");
    return TSV_OK;
}

template <int MODE>
static tsv_status run_verify(const tsv_verify_args* a, RaceParams P, cudaStream_t st) {
    const unsigned scan_blocks = static_cast<unsigned>((a->B + 7) / 8);
    verify_scan_kernel<MODE><<<scan_blocks, 256, 0, st>>>(P);
    TSV_CUDA(cudaGetLastError(), "verify_scan_kernel launch");
    const bool prune = !(a->flags & TSV_VERIFY_NO_PRUNE);
    tsv_status rs;
    if (a->q) rs = prune ? launch_race<MODE, true, true>(P, st) : launch_race<MODE, true, false>(P, st);
    else rs = prune ? launch_race<MODE, false, true>(P, st) : launch_race<MODE, false, false>(P, st);
    TSV_TRY(rs);
    const int64_t units = (MODE == kLazy) ? a->B : a->rows_p;
    TSV_CUDA(launch_pdl(verify_emit_kernel<MODE>, dim3(static_cast<unsigned>((units + 7) / 8)), dim3(256), 0, st, P),
             "verify_emit_kernel launch");
    return TSV_OK;
}

}  // namespace tsv

using namespace tsv;

extern "C" tsv_status tsv_verify_workspace_size(const tsv_verify_args* a, size_t* bytes) {
    TSV_REQUIRE(bytes != nullptr, "tsv_verify_workspace_size: bytes is NULL");
    TSV_TRY(validate(a));
    *bytes = workspace_bytes(a);
    return TSV_OK;
}

extern "C" tsv_status tsv_workspace_clear(void* workspace, size_t bytes, void* stream) {
    if (bytes == 0) return TSV_OK;
    TSV_REQUIRE(workspace != nullptr, "tsv_workspace_clear: workspace is NULL");
    TSV_CUDA(cudaMemsetAsync(workspace, 0, bytes, static_cast<cudaStream_t>(stream)), "cudaMemsetAsync");
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_accept(const tsv_verify_args* a, void* stream) {
    TSV_TRY(validate(a));
    TSV_REQUIRE(a->vocab_offset == 0 && a->vocab == a->vocab_global,
                "tsv_verify_accept: unsharded call needs vocab_offset == 0 and vocab == vocab_global "
                "(use tsv_verify_shard_partial/combine for vocab shards)");
    TSV_TRY(check_device());
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE(a->workspace != nullptr && a->workspace_bytes >= workspace_bytes(a),
                "tsv_verify_accept: workspace too small (%llu < %llu bytes)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)workspace_bytes(a));
    return run_verify<kLazy>(a, make_params(a), static_cast<cudaStream_t>(stream));
}

extern "C" tsv_status tsv_verify_shard_partial(const tsv_verify_args* a, tsv_shard_tuple* tuples_out,
                                               void* stream) {
    TSV_TRY(validate(a));
    TSV_TRY(check_device());
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE(tuples_out != nullptr, "tsv_verify_shard_partial: tuples_out is NULL");
    TSV_REQUIRE(a->workspace != nullptr && a->workspace_bytes >= workspace_bytes(a),
                "tsv_verify_shard_partial: workspace too small (%llu < %llu bytes)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)workspace_bytes(a));
    RaceParams P = make_params(a);
    P.tuples = tuples_out;
    return run_verify<kShard>(a, P, static_cast<cudaStream_t>(stream));
}

extern "C" tsv_status tsv_verify_shard_combine(const tsv_verify_args* a, const tsv_shard_tuple* gathered,
                                               int32_t num_shards, void* stream) {
    TSV_TRY(validate(a));
    TSV_TRY(check_device());
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE(gathered != nullptr, "tsv_verify_shard_combine: gathered is NULL");
    TSV_REQUIRE(num_shards >= 1, "tsv_verify_shard_combine: num_shards < 1");
    RaceParams P = make_params(a);
    const int threads = 256;
    const int64_t blocks = (static_cast<int64_t>(a->B) + (threads / 32) - 1) / (threads / 32);
    verify_shard_combine_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(P, gathered, num_shards, a->rows_p);
    TSV_CUDA(cudaGetLastError(), "verify_shard_combine_kernel launch");
    return TSV_OK;
}
