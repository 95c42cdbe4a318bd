// verify.cu -- rejection-sampling verify/accept on sm_100a (K1 lazy, K1d vocab-shard partial,
// shard combine).  PAPER.md:18 [AD], 493-497 [BG]; readings R1-R9 in DESIGN.md section 3.
//
// Work item = (request, vocab chunk) [lazy] or (request, position, vocab chunk) [shard].
// Each CTA: warp 0 runs the acceptance scan (k_i <= 15 gathers + Philox draws, one
// ballot), then all warps stream the selected row (p, plus q on a rejection) with
// 128-bit loads, drawing one Philox4x32-10 call per float4, and run the exponential
// race with a provably conservative prune test: an element
// whose weight cannot reach the best score seen so far is skipped without its log or
// division; survivors are evaluated exactly (double log, IEEE division) and folded
// into a packed (score, ~index) u64 key.  Chunks of one request combine through a
// self-cleaning per-request slot (atomicMax + arrival counter); the last CTA emits.
#include <stdio.h>

#include "common.cuh"

namespace tsv {

struct Slot {
    unsigned long long key;
    unsigned int count;
    unsigned int pad;
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
    Slot* slots;
    tsv_shard_tuple* tuples;
    int64_t ld;
    uint32_t k0, k1, step;
    int32_t B, k_max, vocab, vocab_offset, vocab_global, chunk, n_chunks;
};

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr float kPruneC = 0x1.fffffap-1f;      // 1 - 3*2^-24 <= (1-2^-23)(1-2^-24)
constexpr float kLbC = 0x1.ffffe0p-1f;         // 1 - 2^-20
constexpr float kMinNormal = 0x1p-126f;

// Lower bound on the exact score RN32(w / E(u)) of an element:
// E <= (-ln u)(1+2^-24) <= ((1-u)/u)(1+2^-24), and rcp.approx is within 2^-22.
__device__ __forceinline__ float race_lower_bound(float w, float omu) {
    const float u = __fsub_rn(1.0f, omu);  // exact
    return __fmul_rd(__fmul_rd(w, u), __fmul_rd(rcp_approx(omu), kLbC));
}

__device__ __forceinline__ float prune_scale(float T) {
    return T >= kMinNormal ? __fmul_rd(T, kPruneC) : 0.0f;
}

// Race over local columns [col_begin, col_end) of one row.  Returns this thread's best
// key (0 = no positive weight seen).  residual: w = max(0, p - q) with q a dense row
// (DENSE_Q) or one-hot at local column xm; else w = max(0, p).  All threads of the CTA
// must call it (uniform trip count; warp-level REDUX inside).
template <bool DENSE_Q, bool PRUNE>
__device__ uint64_t race_chunk(const float* __restrict__ prow, const float* __restrict__ qrow,
                               bool residual, int32_t xm, int32_t col_begin, int32_t col_end,
                               uint32_t vglob_base, uint32_t c1, uint32_t rid, uint32_t step,
                               uint32_t k0, uint32_t k1) {
    const float4* p4 = reinterpret_cast<const float4*>(prow);
    const float4* q4 = reinterpret_cast<const float4*>(qrow);
    const int32_t f_begin = col_begin >> 2;
    const int32_t f_end = (col_end + 3) >> 2;
    const int32_t iters = (f_end - f_begin + kThreads - 1) / kThreads;
    const uint32_t quad_base = vglob_base >> 2;
    const bool use_q = DENSE_Q && residual;

    float T = 0.0f, Tc = 0.0f, Tloc = 0.0f;
    uint64_t best = 0;
    bool has_pend = false;
    float pend_w = 0.0f, pend_omu = 1.0f;
    uint32_t pend_x = 0, pend_v = 0;

    for (int32_t it = 0; it < iters; ++it) {
        const int32_t f = f_begin + it * kThreads + static_cast<int32_t>(threadIdx.x);
        const bool inb = f < f_end;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (inb) {
            a = ldg_stream(p4 + f);
            if (use_q) b = ldg_stream(q4 + f);
        }
        const uint4 r = philox4x32_10(quad_base + static_cast<uint32_t>(f), c1, rid, step, k0, k1);
        const float pv[4] = {a.x, a.y, a.z, a.w};
        const float qv[4] = {b.x, b.y, b.z, b.w};
        const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
        float w[4], omu[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int32_t col = 4 * f + e;
            float we;
            if (residual) {
                float qe = qv[e];
                if (!DENSE_Q) qe = (col == xm) ? 1.0f : 0.0f;
                const float d = __fsub_rn(pv[e], qe);
                we = d > 0.0f ? d : 0.0f;
            } else {
                we = pv[e] > 0.0f ? pv[e] : 0.0f;
            }
            w[e] = (col < col_end) ? we : 0.0f;
            omu[e] = one_minus_u_race(rw[e]);
        }
        if (PRUNE && T == 0.0f) {  // warp-uniform warm-up: seed T from lower bounds
            float lb = 0.0f;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (w[e] > 0.0f) lb = fmaxf(lb, race_lower_bound(w[e], omu[e]));
            Tloc = fmaxf(Tloc, lb);
            T = __uint_as_float(__reduce_max_sync(0xFFFFFFFFu, __float_as_uint(Tloc)));
            Tc = prune_scale(T);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const bool cand = PRUNE ? (w[e] > __fmul_rd(Tc, omu[e])) : (w[e] > 0.0f);
            if (cand) {
                const uint32_t vg = vglob_base + static_cast<uint32_t>(4 * f + e);
                if (!PRUNE) {
                    const uint64_t key = exact_race_key(w[e], rw[e], vg);
                    best = key > best ? key : best;
                } else {
                    Tloc = fmaxf(Tloc, race_lower_bound(w[e], omu[e]));
                    if (has_pend && pend_w > __fmul_rd(Tc, pend_omu)) {
                        const uint64_t key = exact_race_key(pend_w, pend_x, pend_v);
                        best = key > best ? key : best;
                        Tloc = fmaxf(Tloc, __uint_as_float(static_cast<uint32_t>(best >> 32)));
                    }
                    has_pend = true;
                    pend_w = w[e];
                    pend_omu = omu[e];
                    pend_x = rw[e];
                    pend_v = vg;
                }
            }
        }
        if (PRUNE) {
            T = __uint_as_float(__reduce_max_sync(0xFFFFFFFFu, __float_as_uint(Tloc)));
            Tc = prune_scale(T);
        }
    }
    if (PRUNE && has_pend && pend_w > __fmul_rd(Tc, pend_omu)) {
        const uint64_t key = exact_race_key(pend_w, pend_x, pend_v);
        best = key > best ? key : best;
    }
    return best;
}

__device__ __forceinline__ uint64_t block_max_u64(uint64_t v, uint64_t* red /* [kWarps] */) {
    v = warp_max_u64(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        uint64_t t = lane < kWarps ? red[lane] : 0ull;
        t = warp_max_u64(t);
        if (lane == 0) red[0] = t;
    }
    __syncthreads();
    const uint64_t r = red[0];
    __syncthreads();
    return r;
}

struct ScanResult {
    int32_t r0, k, qbase, m, xm, ok;
};

// Acceptance scan (R1-R4): run by warp 0; lane j < k tests draft j.  In shard mode a
// lane only tests drafts this shard owns (own_only) and reports accept/owner bits.
__device__ __forceinline__ void acceptance_scan(const RaceParams& P, int32_t i, ScanResult* out,
                                                uint32_t* accept_bits, uint32_t* owner_bits) {
    const int lane = threadIdx.x & 31;
    const int32_t r0 = P.row_offsets[i];
    const int32_t r1 = P.row_offsets[i + 1];
    const int32_t k = r1 - r0 - 1;
    const int32_t qbase = r0 - i;
    int32_t ok = (k >= 0 && k <= P.k_max && qbase >= 0) ? 1 : 0;
    int32_t x = -1;
    bool bad = false, acc = false, own = false;
    if (ok && lane < k) {
        x = P.drafts[qbase + lane];
        bad = x < 0 || x >= P.vocab_global;
        const int32_t xl = x - P.vocab_offset;
        own = !bad && xl >= 0 && xl < P.vocab;
        if (own) {
            const uint4 rr = philox4x32_10(0u, (kPurposeAccept << 16) | static_cast<uint32_t>(lane),
                                           P.rids[i], P.step, P.k0, P.k1);
            const float u = u_acc_from_word(rr.x);
            const float qx = P.q ? P.q[static_cast<int64_t>(qbase + lane) * P.ld + xl] : 1.0f;
            const float px = P.p[static_cast<int64_t>(r0 + lane) * P.ld + xl];
            acc = __fmul_rn(u, qx) < px;  // strict; NaN rejects
        }
    }
    const uint32_t badm = __ballot_sync(0xFFFFFFFFu, bad);
    const uint32_t accm = __ballot_sync(0xFFFFFFFFu, acc);
    const uint32_t ownm = __ballot_sync(0xFFFFFFFFu, own);
    if (badm) ok = 0;
    const uint32_t kmask = (ok && k > 0) ? ((1u << k) - 1u) : 0u;
    const uint32_t rej = ~accm & kmask;
    const int32_t m = rej ? (__ffs(rej) - 1) : (ok ? k : 0);
    const int32_t xm = __shfl_sync(0xFFFFFFFFu, x, m & 31);
    if (lane == 0) {
        out->r0 = r0;
        out->k = k;
        out->qbase = qbase;
        out->m = m;
        out->xm = (m < k) ? xm : -1;
        out->ok = ok | (badm ? 2 : 0);
        if (accept_bits) *accept_bits = accm & kmask;
        if (owner_bits) *owner_bits = ownm & kmask;
    }
}

__device__ __forceinline__ void report(int32_t* devstatus, uint32_t bits) {
    if (devstatus && bits) atomicOr(reinterpret_cast<unsigned int*>(devstatus), bits);
}

// Emit (R1-R4 step 4): lanes j <= k_max of one warp.
__device__ __forceinline__ void emit(const RaceParams& P, int32_t i, int32_t qbase, int32_t m,
                                     int32_t t) {
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

// ------------------------------------------------------------------------- lazy (1 GPU)
template <bool DENSE_Q, bool PRUNE>
__global__ void __launch_bounds__(kThreads) verify_lazy_kernel(const RaceParams P) {
    __shared__ ScanResult s;
    __shared__ uint64_t red[kWarps];
    __shared__ int s_last;
    const int32_t i = blockIdx.x / P.n_chunks;
    const int32_t c = blockIdx.x - i * P.n_chunks;
    if (threadIdx.x < 32) acceptance_scan(P, i, &s, nullptr, nullptr);
    __syncthreads();
    const ScanResult sc = s;
    if (sc.ok != 1) {  // bad k (2: BAD_K) or bad draft token
        if (c == 0 && threadIdx.x < 32) {
            emit(P, i, 0, -1, -1);
            if (threadIdx.x == 0)
                report(P.devstatus, (sc.ok & 2) ? TSV_DEVSTATUS_BAD_TOKEN : TSV_DEVSTATUS_BAD_K);
        }
        return;
    }
    const bool residual = sc.m < sc.k;
    const float* prow = P.p + static_cast<int64_t>(sc.r0 + sc.m) * P.ld;
    const float* qrow = (DENSE_Q && residual) ? P.q + static_cast<int64_t>(sc.qbase + sc.m) * P.ld : nullptr;
    const int32_t xm_local = residual ? sc.xm - P.vocab_offset : -1;
    const int32_t col_begin = c * P.chunk;
    const int32_t col_end = min(P.vocab, col_begin + P.chunk);
    const uint32_t c1 = (kPurposeRace << 16) | static_cast<uint32_t>(sc.m);
    const uint32_t rid = P.rids[i];
    uint64_t best = race_chunk<DENSE_Q, PRUNE>(prow, qrow, residual, xm_local, col_begin, col_end,
                                               static_cast<uint32_t>(P.vocab_offset), c1, rid,
                                               P.step, P.k0, P.k1);
    best = block_max_u64(best, red);
    if (P.n_chunks > 1) {
        if (threadIdx.x == 0) {
            Slot* sl = P.slots + i;
            atomicMax(&sl->key, static_cast<unsigned long long>(best));
            __threadfence();
            const unsigned int prev = atomicAdd(&sl->count, 1u);
            int last = 0;
            if (prev == static_cast<unsigned int>(P.n_chunks - 1)) {
                best = atomicExch(&sl->key, 0ull);  // final value; leaves the slot clean
                atomicExch(&sl->count, 0u);
                last = 1;
            }
            s_last = last;
            red[0] = best;
        }
        __syncthreads();
        if (!s_last) return;
        best = red[0];
    }
    if (best == 0 && residual) {  // residual identically zero: fall back to p_m (R5)
        uint64_t fb = race_chunk<DENSE_Q, PRUNE>(prow, nullptr, false, -1, 0, P.vocab,
                                                 static_cast<uint32_t>(P.vocab_offset), c1, rid,
                                                 P.step, P.k0, P.k1);
        best = block_max_u64(fb, red);
    }
    if (threadIdx.x < 32) {
        const int32_t t = best ? key_index(best) : -1;
        emit(P, i, sc.qbase, sc.m, t);
        if (threadIdx.x == 0 && !best) report(P.devstatus, TSV_DEVSTATUS_NO_WEIGHT);
    }
}

// ------------------------------------------------------------------ vocab-shard partial
// Item = (request i, position j, chunk c); rows j > k_i exit.  Dense: every row of
// every request is raced over this shard's columns (the one-round exchange, R-shard).
template <bool DENSE_Q, bool PRUNE>
__global__ void __launch_bounds__(kThreads) verify_shard_partial_kernel(const RaceParams P) {
    __shared__ ScanResult s;
    __shared__ uint64_t red[kWarps];
    __shared__ uint32_t s_acc, s_own;
    __shared__ int s_last;
    const int32_t per_req = (P.k_max + 1) * P.n_chunks;
    const int32_t i = blockIdx.x / per_req;
    const int32_t rem = blockIdx.x - i * per_req;
    const int32_t j = rem / P.n_chunks;
    const int32_t c = rem - j * P.n_chunks;
    if (threadIdx.x < 32) acceptance_scan(P, i, &s, &s_acc, &s_own);
    __syncthreads();
    const ScanResult sc = s;
    if (sc.ok != 1 || j > sc.k) return;  // invalid requests are flagged by the combine
    const int32_t row = sc.r0 + j;
    if (c == 0 && threadIdx.x == 0) {
        uint32_t flag = 0;
        if (j < sc.k) flag = ((s_acc >> j) & 1u) | (((s_own >> j) & 1u) << 1);
        P.tuples[row].flag = flag;
        P.tuples[row].pad = 0;
    }
    const bool residual = j < sc.k;
    int32_t xj = -1;
    if (residual && !DENSE_Q) xj = P.drafts[sc.qbase + j] - P.vocab_offset;
    const float* prow = P.p + static_cast<int64_t>(row) * P.ld;
    const float* qrow = (DENSE_Q && residual) ? P.q + static_cast<int64_t>(sc.qbase + j) * P.ld : nullptr;
    const int32_t col_begin = c * P.chunk;
    const int32_t col_end = min(P.vocab, col_begin + P.chunk);
    const uint32_t c1 = (kPurposeRace << 16) | static_cast<uint32_t>(j);
    const uint32_t rid = P.rids[i];
    uint64_t best = race_chunk<DENSE_Q, PRUNE>(prow, qrow, residual, xj, col_begin, col_end,
                                               static_cast<uint32_t>(P.vocab_offset), c1, rid,
                                               P.step, P.k0, P.k1);
    best = block_max_u64(best, red);
    if (P.n_chunks > 1) {
        if (threadIdx.x == 0) {
            Slot* sl = P.slots + row;
            atomicMax(&sl->key, static_cast<unsigned long long>(best));
            __threadfence();
            const unsigned int prev = atomicAdd(&sl->count, 1u);
            int last = 0;
            if (prev == static_cast<unsigned int>(P.n_chunks - 1)) {
                best = atomicExch(&sl->key, 0ull);
                atomicExch(&sl->count, 0u);
                last = 1;
            }
            s_last = last;
            red[0] = best;
        }
        __syncthreads();
        if (!s_last) return;
        best = red[0];
    }
    uint64_t fb = 0;
    if (best == 0 && residual) {
        fb = race_chunk<DENSE_Q, PRUNE>(prow, nullptr, false, -1, 0, P.vocab,
                                        static_cast<uint32_t>(P.vocab_offset), c1, rid, P.step,
                                        P.k0, P.k1);
        fb = block_max_u64(fb, red);
    }
    if (threadIdx.x == 0) {
        P.tuples[row].key = best;
        P.tuples[row].fb_key = fb;
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
static int32_t auto_chunk(const tsv_verify_args* a) {
    if (a->chunk > 0) return a->chunk;
    return 8192;
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
    TSV_REQUIRE(a->chunk == 0 || (a->chunk > 0 && a->chunk % 1024 == 0), "tsv_verify: chunk must be 0 or a multiple of 1024");
    return TSV_OK;
}

static RaceParams make_params(const tsv_verify_args* a, int32_t chunk) {
    RaceParams P;
    P.p = a->p;
    P.q = a->q;
    P.row_offsets = a->row_offsets;
    P.drafts = a->draft_tokens;
    P.rids = a->request_ids;
    P.num_accepted = a->num_accepted;
    P.out_tokens = a->out_tokens;
    P.devstatus = a->device_status;
    P.slots = reinterpret_cast<Slot*>(a->workspace);
    P.tuples = nullptr;
    P.ld = a->ld;
    P.k0 = static_cast<uint32_t>(a->seed & 0xFFFFFFFFull);
    P.k1 = static_cast<uint32_t>(a->seed >> 32);
    P.step = a->step;
    P.B = a->B;
    P.k_max = a->k_max;
    P.vocab = a->vocab;
    P.vocab_offset = a->vocab_offset;
    P.vocab_global = a->vocab_global;
    P.chunk = chunk;
    P.n_chunks = (a->vocab + chunk - 1) / chunk;
    return P;
}

}  // namespace tsv

using namespace tsv;

extern "C" tsv_status tsv_verify_workspace_size(const tsv_verify_args* a, size_t* bytes) {
    TSV_REQUIRE(bytes != nullptr, "tsv_verify_workspace_size: bytes is NULL");
    TSV_TRY(validate(a));
    *bytes = static_cast<size_t>(a->rows_p > a->B ? a->rows_p : a->B) * sizeof(Slot);
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
    const int32_t chunk = auto_chunk(a);
    RaceParams P = make_params(a, chunk);
    if (P.n_chunks > 1) {
        TSV_REQUIRE(a->workspace != nullptr && a->workspace_bytes >= static_cast<uint64_t>(a->B) * sizeof(Slot),
                    "tsv_verify_accept: workspace too small (%llu < %llu bytes)",
                    (unsigned long long)a->workspace_bytes, (unsigned long long)(a->B * sizeof(Slot)));
    }
    const int64_t grid = static_cast<int64_t>(a->B) * P.n_chunks;
    TSV_REQUIRE(grid < (1ll << 31), "tsv_verify_accept: grid too large");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool prune = !(a->flags & TSV_VERIFY_NO_PRUNE);
    if (a->q) {
        if (prune) verify_lazy_kernel<true, true><<<grid, kThreads, 0, st>>>(P);
        else verify_lazy_kernel<true, false><<<grid, kThreads, 0, st>>>(P);
    } else {
        if (prune) verify_lazy_kernel<false, true><<<grid, kThreads, 0, st>>>(P);
        else verify_lazy_kernel<false, false><<<grid, kThreads, 0, st>>>(P);
    }
    TSV_CUDA(cudaGetLastError(), "verify_lazy_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_shard_partial(const tsv_verify_args* a, tsv_shard_tuple* tuples_out,
                                               void* stream) {
    TSV_TRY(validate(a));
    TSV_TRY(check_device());
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE(tuples_out != nullptr, "tsv_verify_shard_partial: tuples_out is NULL");
    const int32_t chunk = auto_chunk(a);
    RaceParams P = make_params(a, chunk);
    P.tuples = tuples_out;
    if (P.n_chunks > 1) {
        TSV_REQUIRE(a->workspace != nullptr && a->workspace_bytes >= static_cast<uint64_t>(a->rows_p) * sizeof(Slot),
                    "tsv_verify_shard_partial: workspace too small");
    }
    const int64_t grid = static_cast<int64_t>(a->B) * (a->k_max + 1) * P.n_chunks;
    TSV_REQUIRE(grid < (1ll << 31), "tsv_verify_shard_partial: grid too large");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool prune = !(a->flags & TSV_VERIFY_NO_PRUNE);
    if (a->q) {
        if (prune) verify_shard_partial_kernel<true, true><<<grid, kThreads, 0, st>>>(P);
        else verify_shard_partial_kernel<true, false><<<grid, kThreads, 0, st>>>(P);
    } else {
        if (prune) verify_shard_partial_kernel<false, true><<<grid, kThreads, 0, st>>>(P);
        else verify_shard_partial_kernel<false, false><<<grid, kThreads, 0, st>>>(P);
    }
    TSV_CUDA(cudaGetLastError(), "verify_shard_partial_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_shard_combine(const tsv_verify_args* a, const tsv_shard_tuple* gathered,
                                               int32_t num_shards, void* stream) {
    TSV_TRY(validate(a));
    TSV_TRY(check_device());
    if (a->B == 0) return TSV_OK;
    TSV_REQUIRE(gathered != nullptr, "tsv_verify_shard_combine: gathered is NULL");
    TSV_REQUIRE(num_shards >= 1, "tsv_verify_shard_combine: num_shards < 1");
    RaceParams P = make_params(a, auto_chunk(a));
    const int threads = 256;
    const int64_t blocks = (static_cast<int64_t>(a->B) + (threads / 32) - 1) / (threads / 32);
    verify_shard_combine_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(P, gathered, num_shards, a->rows_p);
    TSV_CUDA(cudaGetLastError(), "verify_shard_combine_kernel launch");
    return TSV_OK;
}
