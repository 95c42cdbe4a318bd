// goodput.cuh -- ArgMaxGoodput and the acceptance update as CTA-wide device routines, shared by
// the standalone kernels (goodput.cu) and the fused kernels (lookup + choose-k in lookup.cu,
// verify emit + update in verify.cu).  See goodput.cu for the paper passages and readings.
#pragma once

#include "common.cuh"
#include "p2p.cuh"

namespace tsv {

constexpr int kGpThreads = 256;
constexpr int kGpWarps = kGpThreads / 32;
constexpr int kGpMaxK = TSV_MAX_K + 1;

// Exact warp sum of int64 values with three redux.sync adds: 21-bit limbs (the top one
// signed) whose 32-lane sums fit in 32 bits; recombined mod 2^64, i.e. exact whenever the
// true sum fits in int64.
__device__ __forceinline__ long long warp_sum_i64(long long v) {
    const unsigned l0 = static_cast<unsigned>(v) & 0x1FFFFFu;
    const unsigned l1 = static_cast<unsigned>(v >> 21) & 0x1FFFFFu;
    const int l2 = static_cast<int>(v >> 42);
    const unsigned s0 = __reduce_add_sync(0xFFFFFFFFu, l0);
    const unsigned s1 = __reduce_add_sync(0xFFFFFFFFu, l1);
    const int s2 = __reduce_add_sync(0xFFFFFFFFu, l2);
    const unsigned long long r = static_cast<unsigned long long>(s0) + (static_cast<unsigned long long>(s1) << 21) +
                                 (static_cast<unsigned long long>(static_cast<long long>(s2)) << 42);
    return static_cast<long long>(r);
}

__device__ __forceinline__ double fwd_time(const tsv_latency_model& m, double n_ctx, double n_batched) {
    return __fma_rn(m.batched_ms_per_tok, n_batched, __fma_rn(m.ctx_ms_per_tok, n_ctx, m.fixed_ms));
}

struct ChooseArgs {
    const double* alpha;
    const int32_t* ctx_len;
    const int32_t* cap;
    int32_t* k_out;
    double* goodput_out;
    int32_t* k_per_request;
    tsv_latency_model target, draft;
    double pld_cost_ms;
    long long kv_free;
    int32_t alpha_per_request, B, k_max, policy;
    const uint32_t* alpha_ready;  // nullable: wait for *alpha_ready == 1 before reading alpha (fused lookup)
    int32_t* devstatus;           // TSV_DEVSTATUS_WAIT_TIMEOUT (nullable)
};

struct UpdateArgs {
    double* alpha;
    const int32_t* num_accepted;
    const int32_t* row_offsets;
    double decay;
    int32_t per_request, B, estimator;
    // request-sharded global alpha: the (sum m, sum t) pair is summed over the
    // ranks through peer memory (p2p.cuh) before the EWMA; every rank applies the same update
    int32_t use_p2p;
    int32_t* devstatus;  // TSV_DEVSTATUS_P2P_TIMEOUT (nullable)
    P2PView p2p;
    // nullable (tsv_verify_accept_update_ex): set to 1 with release semantics once alpha is written, so
    // a kernel that starts before this call completes (TSV_VERIFY_EARLY_TRIGGER) can wait for alpha
    uint32_t* alpha_ready;
};

// alpha is written (by this thread, or by this CTA before a __syncthreads): publish it
__device__ __forceinline__ void signal_alpha_ready(uint32_t* flag) {
    if (flag) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(1u) : "memory");
    }
}

// Wait (bounded, %globaltimer) until *flag == 1 with acquire semantics; TSV_DEVSTATUS_WAIT_TIMEOUT if it
// never comes (the producer is not running: a contract violation), instead of hanging.
__device__ __forceinline__ void wait_alpha_ready(const uint32_t* flag, int32_t* devstatus) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v == 1u) return;
    const unsigned long long t0 = global_ns();
    uint32_t n = 0;
    while (v != 1u) {
        __nanosleep(64);
        if ((++n & 255u) == 0 && global_ns() - t0 > TSV_P2P_TIMEOUT_NS) {
            report(devstatus, TSV_DEVSTATUS_WAIT_TIMEOUT);
            return;
        }
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    }
}

// Batch sums of ArgMaxGoodput, exact int64 (fixed point 2^-32 for the token sums):
//   L[k] = sum_i rint(2^32 l(alpha_i, min(k, cap_i))),  N[k] = sum_i min(k, cap_i),
//   c[0] = sum_i ctx_len_i,  c[1] = sum over cap_i > 0 of ctx_len_i,  c[2] = #{cap_i > 0},
//   c[3] = B.
// Sums over disjoint request sets add up to the sums of their union (request-sharded mode).
struct GpTotals {  // per lane k of warp 0: L[k], N[k]; every lane: c[0..3]
    long long L, N, c0, c1, c2, c3;
};

// CTA-wide (all kGpThreads threads call); the result is valid in warp 0.
// Each thread accumulates its requests for every candidate k (the Horner recurrence
// l(a, j+1) = fma(a, l(a, j), 1) advanced once each time min(k, cap_i) grows, op-for-op a
// fresh evaluation); warp sums are exact redux.sync limb sums, then one shared-memory step.
constexpr int kGpCapCache = 4;  // caps kept in registers for k_i = min(k*, cap_i) (B <= 4 NT)
// Global alpha: every request's term depends only on j_i = clamp(cap_i, 0, k_max), so the batch sums
// follow from the histogram n_j of the j_i:  L[k] = sum_j n_j rint(2^32 l(alpha, min(k, j))) and
// N[k] = sum_j n_j min(k, j) -- the same exact int64 values as summing the requests' terms one by one
// (integer addition is exact and order-free; each term is the same function of (alpha, min(k, j_i))).
// l(alpha, j) is evaluated once per j by warp 0 with the same Horner recurrence.  The histogram needs
// one redux per bin instead of a Horner chain and 64-bit conversions per request.
#ifndef TSV_GP_HISTOGRAM
#define TSV_GP_HISTOGRAM 1
#endif
// The histogram's batch sums (one warp, lane j holding n_j for j <= k_max): fix_j = rint(2^32 l(alpha, j))
// by the Horner recurrence from 1.0 (j steps), then lane k: L[k] = sum_{j<k} n_j fix_j + (sum_{j>=k} n_j)
// fix_k and N[k] = sum_j n_j min(k, j).
__device__ __forceinline__ void gp_hist_tail(GpTotals& t, long long nj, double a, int32_t k_max, int lane) {
    double l = 1.0;
    for (int s = 0; s < lane && s < k_max; ++s) l = __fma_rn(a, l, 1.0);
    const long long fix_j = __double2ll_rn(l * 0x1p32);
    long long Lk = 0, Nk = 0, tail = 0;
    for (int j = 0; j <= k_max; ++j) {
        const long long n_ = __shfl_sync(0xFFFFFFFFu, nj, j);
        const long long f_ = __shfl_sync(0xFFFFFFFFu, fix_j, j);
        if (j < lane) {
            Lk += n_ * f_;
            Nk += n_ * j;
        } else {
            tail += n_;
        }
    }
    if (lane <= k_max) {
        t.L = Lk + tail * fix_j;
        t.N = Nk + tail * lane;
    }
}

// The same sums from ONE warp (global alpha): no shared memory, no barrier.  Lane l takes requests l,
// l + 32, ...; its bin counts are 8-bit fields of two 64-bit words (<= 255 requests per lane: B <= 8160),
// summed over the warp one bin per REDUX; the context sums are exact int64 warp sums.  Identical integers
// to gp_sums_block_hist (integer addition is exact and order-free), so identical k* and goodput bits.
constexpr int kGpWarpMaxB = 32 * 255;
constexpr int kGpWarpCaps = 8;  // caps kept in registers for k_i = min(k*, cap_i)
__device__ __forceinline__ GpTotals gp_sums_warp(const ChooseArgs& A, int32_t (&cap_cache)[kGpWarpCaps]) {
    const int lane = threadIdx.x & 31;
    const int32_t B = A.B, k_max = A.k_max;
    const double a = __ldcg(A.alpha);  // every lane (broadcast): the Horner recurrence is per lane
    long long n_ctx = 0, n_ctx_spec = 0;
    uint32_t b_spec = 0;
    unsigned long long f_lo = 0ull, f_hi = 0ull;  // bins 0-7 / 8-15, 8 bits each
    auto take = [&](int32_t ci, int32_t cl) {
        n_ctx += cl;
        if (ci > 0) {
            n_ctx_spec += cl;
            b_spec += 1;
        }
        const int32_t j = ci < 0 ? 0 : (ci > k_max ? k_max : ci);
        if (j < 8) f_lo += 1ull << (8 * j);
        else f_hi += 1ull << (8 * (j - 8));
    };
    // the first 32 kGpWarpCaps requests: every load issued before any is used (one round trip)
    int32_t cls[kGpWarpCaps];
#pragma unroll
    for (int r = 0; r < kGpWarpCaps; ++r) {
        const int32_t i = r * 32 + lane;
        cap_cache[r] = i < B ? __ldcg(A.cap + i) : 0;
        cls[r] = i < B ? __ldcg(A.ctx_len + i) : 0;
    }
#pragma unroll
    for (int r = 0; r < kGpWarpCaps; ++r)
        if (r * 32 + lane < B) take(cap_cache[r], cls[r]);
    for (int32_t i = kGpWarpCaps * 32 + lane; i < B; i += 32) take(__ldcg(A.cap + i), __ldcg(A.ctx_len + i));
    long long nj = 0;  // lane j: n_j
#pragma unroll
    for (int b = 0; b < kGpMaxK; ++b) {
        if (b <= k_max) {
            const uint32_t field = static_cast<uint32_t>(((b < 8 ? f_lo : f_hi) >> (8 * (b & 7))) & 0xFFull);
            const uint32_t h = __reduce_add_sync(0xFFFFFFFFu, field);
            if (lane == b) nj = h;
        }
    }
    GpTotals t = {0, 0, warp_sum_i64(n_ctx), warp_sum_i64(n_ctx_spec),
                  static_cast<long long>(__reduce_add_sync(0xFFFFFFFFu, b_spec)), static_cast<long long>(B)};
    gp_hist_tail(t, nj, a, k_max, lane);
    return t;
}

template <int NT>
__device__ __forceinline__ GpTotals gp_sums_block_hist(const ChooseArgs& A, int32_t* cap_cache) {
    constexpr int NW = NT / 32;
    __shared__ uint32_t sH[NW][kGpMaxK];
    __shared__ long long sC[NW][3];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t B = A.B, k_max = A.k_max;
    uint32_t cnt[kGpMaxK];
#pragma unroll
    for (int j = 0; j < kGpMaxK; ++j) cnt[j] = 0;
    long long n_ctx = 0, n_ctx_spec = 0;
    uint32_t b_spec = 0;  // #{cap_i > 0} (not n_0's complement: with k_max = 0 every j_i is 0)
    const double a = warp == 0 ? __ldcg(A.alpha) : 0.0;  // issued with the caps: one round trip for both
    int slot = 0;
    for (int32_t i = threadIdx.x; i < B; i += NT, ++slot) {
        const int32_t ci = __ldcg(A.cap + i);
        if (cap_cache && slot < kGpCapCache) cap_cache[slot] = ci;
        const int32_t cl = __ldcg(A.ctx_len + i);
        n_ctx += cl;
        if (ci > 0) {
            n_ctx_spec += cl;
            b_spec += 1;
        }
        const int32_t j = ci < 0 ? 0 : (ci > k_max ? k_max : ci);
#pragma unroll
        for (int b = 0; b < kGpMaxK; ++b) cnt[b] += (b == j) ? 1u : 0u;
    }
#pragma unroll
    for (int b = 0; b < kGpMaxK; ++b) {
        if (b <= k_max) {
            const uint32_t h = __reduce_add_sync(0xFFFFFFFFu, cnt[b]);
            if (lane == 0) sH[warp][b] = h;
        }
    }
    n_ctx = warp_sum_i64(n_ctx);
    n_ctx_spec = warp_sum_i64(n_ctx_spec);
    const uint32_t b_spec_w = __reduce_add_sync(0xFFFFFFFFu, b_spec);
    if (lane == 0) {
        sC[warp][0] = n_ctx;
        sC[warp][1] = n_ctx_spec;
        sC[warp][2] = b_spec_w;
    }
    __syncthreads();
    GpTotals t = {0, 0, 0, 0, 0, static_cast<long long>(B)};
    if (warp == 0) {
        long long nj = 0;  // lane j: n_j
        if (lane <= k_max)
#pragma unroll
            for (int w = 0; w < NW; ++w) nj += sH[w][lane];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            t.c0 += sC[w][0];
            t.c1 += sC[w][1];
            t.c2 += sC[w][2];
        }
        gp_hist_tail(t, nj, a, k_max, lane);
    }
    return t;
}

template <int NT = kGpThreads>
__device__ __forceinline__ GpTotals gp_sums_block(const ChooseArgs& A, int32_t* cap_cache = nullptr) {
    if (TSV_GP_HISTOGRAM && !A.alpha_per_request) return gp_sums_block_hist<NT>(A, cap_cache);
    constexpr int NW = NT / 32;
    __shared__ long long sL[NW][kGpMaxK];
    __shared__ long long sN[NW][kGpMaxK];
    __shared__ long long sC[NW][3];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t B = A.B, k_max = A.k_max;
    long long Lk[kGpMaxK];
    uint32_t Nk[kGpMaxK];  // sum_i min(k, cap_i) <= 15 B
#pragma unroll
    for (int k = 0; k < kGpMaxK; ++k) Lk[k] = 0, Nk[k] = 0;
    long long n_ctx = 0, n_ctx_spec = 0;
    uint32_t b_spec = 0;
    const double a_glob = A.alpha_per_request ? 0.0 : __ldcg(A.alpha);
    int slot = 0;
    for (int32_t i = threadIdx.x; i < B; i += NT, ++slot) {
        const double a = A.alpha_per_request ? __ldcg(A.alpha + i) : a_glob;
        const int32_t ci = __ldcg(A.cap + i);
        if (cap_cache && slot < kGpCapCache) cap_cache[slot] = ci;
        const int32_t cl = __ldcg(A.ctx_len + i);
        n_ctx += cl;
        if (ci > 0) {
            n_ctx_spec += cl;
            b_spec += 1;
        }
        double l = 1.0;
        long long fix = __double2ll_rn(l * 0x1p32);
#pragma unroll
        for (int k = 0; k < kGpMaxK; ++k) {
            if (k <= k_max) {
                if (k >= 1 && k <= ci) {
                    l = __fma_rn(a, l, 1.0);
                    fix = __double2ll_rn(l * 0x1p32);
                }
                Lk[k] += fix;
                Nk[k] += static_cast<uint32_t>(k <= ci ? k : (ci > 0 ? ci : 0));
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kGpMaxK; ++k) {
        if (k <= k_max) {
            const long long l = warp_sum_i64(Lk[k]);
            const long long n = __reduce_add_sync(0xFFFFFFFFu, Nk[k]);
            if (lane == 0) {
                sL[warp][k] = l;
                sN[warp][k] = n;
            }
        }
    }
    n_ctx = warp_sum_i64(n_ctx);
    n_ctx_spec = warp_sum_i64(n_ctx_spec);
    const long long b_spec_w = __reduce_add_sync(0xFFFFFFFFu, b_spec);
    if (lane == 0) {
        sC[warp][0] = n_ctx;
        sC[warp][1] = n_ctx_spec;
        sC[warp][2] = b_spec_w;
    }
    __syncthreads();
    GpTotals t = {0, 0, 0, 0, 0, static_cast<long long>(B)};
    if (warp == 0) {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            t.c0 += sC[w][0];
            t.c1 += sC[w][1];
            t.c2 += sC[w][2];
        }
        if (lane <= k_max) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                t.L += sL[w][lane];
                t.N += sN[w][lane];
            }
        }
    }
    return t;
}

// Warp 0 only: lane k evaluates T(k) and G(k) from the totals, lane 0 runs Listing 2's
// strict-'>' scan over k = 0..k_max (k = 0 included, reading R12); writes k_out and
// goodput_out; returns k* in every lane.
__device__ __forceinline__ int gp_argmax_warp(const ChooseArgs& A, const GpTotals& t) {
    const int lane = threadIdx.x & 31;
    const int32_t k_max = A.k_max;
    double g = -1.0;
    bool valid = false;
    if (lane <= k_max) {
        const long long n_batched = t.N + t.c3;
        if (!(lane > 0 && A.kv_free >= 0 && n_batched > A.kv_free)) {  // Listing 2 line 5: OOM -> skip
            const double t_target = fwd_time(A.target, static_cast<double>(t.c0), static_cast<double>(n_batched));
            double t_draft;
            if (A.policy == TSV_POLICY_PLD)
                t_draft = A.pld_cost_ms;
            else
                t_draft = lane > 0 ? __dmul_rn(static_cast<double>(lane),
                                               fwd_time(A.draft, static_cast<double>(t.c1), static_cast<double>(t.c2)))
                                   : 0.0;
            g = __ddiv_rn(__dmul_rn(static_cast<double>(t.L), 0x1p-32), __dadd_rn(t_target, t_draft));
            valid = true;
        }
        if (A.goodput_out) A.goodput_out[lane] = g;
    }
    // Listing 2: max_goodput = -1; for k: if goodput > max_goodput: take k (strict >)
    double max_goodput = -1.0;
    int best_k = 0;
    for (int k = 0; k <= k_max; ++k) {
        const double gk = __shfl_sync(0xFFFFFFFFu, g, k);
        const bool vk = __shfl_sync(0xFFFFFFFFu, valid, k);
        if (vk && gk > max_goodput) {
            max_goodput = gk;
            best_k = k;
        }
    }
    if (lane == 0) *A.k_out = best_k;
    return best_k;
}

// k_i = min(k*, cap_i) for this CTA's requests (all threads; k* from shared memory; caps from
// the registers of gp_sums_block when given, else reloaded).
template <int NT = kGpThreads>
__device__ __forceinline__ void gp_write_k_per_request(const ChooseArgs& A, int kb, const int32_t* cap_cache = nullptr) {
    int slot = 0;
    for (int32_t i = threadIdx.x; i < A.B; i += NT, ++slot) {
        const int32_t ci = (cap_cache && slot < kGpCapCache) ? cap_cache[slot] : __ldcg(A.cap + i);
        const int32_t ki = kb < ci ? kb : ci;
        A.k_per_request[i] = ki < 0 ? 0 : ki;
    }
}

// ArgMaxGoodput over one CTA of kGpThreads threads (all threads must call).  Inputs are read
// with ld.global.cg so values written by other CTAs of a fused kernel are seen.
// ArgMaxGoodput by warp 0 alone (global alpha, B <= kGpWarpMaxB; the other warps return): the batch sums,
// Listing 2 and k_i = min(k*, cap_i), with no shared memory or barrier on the chain.  Used for one-warp CTAs
// and small batches (choose_k_block).
#ifndef TSV_GP_WARP
#define TSV_GP_WARP 1
#endif
__device__ __forceinline__ bool choose_k_warp_ok(const ChooseArgs& A) {
    return TSV_GP_WARP && TSV_GP_HISTOGRAM && !A.alpha_per_request && A.B <= kGpWarpMaxB;
}
__device__ __forceinline__ void choose_k_warp(const ChooseArgs& A) {
    int32_t caps[kGpWarpCaps];
    const GpTotals t = gp_sums_warp(A, caps);
    const int kb = gp_argmax_warp(A, t);
    if (A.k_per_request) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int r = 0; r < kGpWarpCaps; ++r) {
            const int32_t i = r * 32 + lane;
            if (i < A.B) {
                const int32_t ki = kb < caps[r] ? kb : caps[r];
                A.k_per_request[i] = ki < 0 ? 0 : ki;
            }
        }
        for (int32_t i = kGpWarpCaps * 32 + lane; i < A.B; i += 32) {
            const int32_t ci = __ldcg(A.cap + i);
            const int32_t ki = kb < ci ? kb : ci;
            A.k_per_request[i] = ki < 0 ? 0 : ki;
        }
    }
}

template <int NT = kGpThreads>
__device__ __forceinline__ void choose_k_block(const ChooseArgs& A) {
    // one warp when the CTA is one warp anyway (the batched kernel: config 5 7.9 vs 9.6 us) or the batch is
    // small; for B = 256 on 256 threads the eight warps' parallel loads and sums win (21.1 vs 21.45 us step)
    if (choose_k_warp_ok(A) && (NT == 32 || A.B <= 64)) {
        if ((threadIdx.x >> 5) == 0) choose_k_warp(A);
        return;
    }
    __shared__ int s_best;
    int32_t caps[kGpCapCache];
    const GpTotals t = gp_sums_block<NT>(A, caps);
    if ((threadIdx.x >> 5) == 0) {
        const int kb = gp_argmax_warp(A, t);
        if (threadIdx.x == 0) s_best = kb;
    }
    if (A.k_per_request) {
        __syncthreads();
        gp_write_k_per_request<NT>(A, s_best, caps);
    }
}

// alpha' = fma(d, alpha - r, r), r = RN64(sum_m / sum_t); no update when sum_t == 0.
__device__ __forceinline__ void ewma_apply(double* alpha, long long sum_m, long long sum_t, double decay) {
    if (sum_t > 0) {
        const double r = __ddiv_rn(static_cast<double>(sum_m), static_cast<double>(sum_t));
        *alpha = __fma_rn(decay, __dsub_rn(*alpha, r), r);
    }
}

// UpdateGlobalAcceptance over one CTA of kGpThreads threads (all threads must call).
// Global mode: the exact int64 sums (sum_m, sum_t) land in thread 0 and are either applied
// (sums_out == nullptr) or written to sums_out[0..1] (request-sharded partial).
__device__ __forceinline__ void update_block(const UpdateArgs& A, long long* sums_out = nullptr) {
    __shared__ long long red[kGpWarps][2];
    long long sm = 0, stt = 0;
    for (int32_t i = threadIdx.x; i < A.B; i += kGpThreads) {
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
        red[warp][0] = sm;
        red[warp][1] = stt;
    }
    __syncthreads();
    __shared__ long long s_ab[2];
    if (threadIdx.x == 0) {
        long long a = 0, b = 0;
#pragma unroll
        for (int w = 0; w < kGpWarps; ++w) {
            a += red[w][0];
            b += red[w][1];
        }
        if (sums_out) {
            sums_out[0] = a;
            sums_out[1] = b;
        } else if (!A.use_p2p) {
            ewma_apply(A.alpha, a, b, A.decay);
            signal_alpha_ready(A.alpha_ready);
        }
        s_ab[0] = a;
        s_ab[1] = b;
    }
    if (A.use_p2p && !sums_out) {  // the ranks' pairs summed over peer memory, then the same EWMA everywhere
        __syncthreads();
        p2p_allreduce_block(s_ab, 2, A.p2p, A.devstatus);
        if (threadIdx.x == 0) {
            ewma_apply(A.alpha, s_ab[0], s_ab[1], A.decay);
            signal_alpha_ready(A.alpha_ready);
        }
    }
}

}  // namespace tsv
