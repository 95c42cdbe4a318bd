// goodput.cu -- goodput k-selector (K3) and acceptance-rate update (K4) on sm_100a.
//
// ArgMaxGoodput (Listing 2, PAPER.md:256-270 [AD]) with Eq. goodput,
// Eq. batch-latency, Eq. forward-time,
// T_draft = s * T_fwd and the batch sum of Eq. gen_len
// (PAPER.md:133-143); UpdateGlobalAcceptance (Listing 1) with the
// moving average of PAPER.md:131-132.  Readings R11-R19.
//
// Exactness by construction: l(alpha, j) is the Horner recurrence
// l_j = fma(alpha, l_{j-1}, 1), identical op for op to a fresh evaluation; each
// request's l is quantised once to 2^-32 fixed point (rint) and summed in int64,
// so the batch sums are exact and independent of reduction order, block shape or
// the number of ranks that contribute partial sums.
#include "common.cuh"

namespace tsv {

constexpr int kGpThreads = 256;
constexpr int kGpWarps = kGpThreads / 32;
constexpr int kGpMaxK = TSV_MAX_K + 1;

__device__ __forceinline__ long long warp_sum_i64(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

__device__ __forceinline__ double fwd_time(const tsv_latency_model& m, double n_ctx, double n_batched) {
    return __fma_rn(m.batched_ms_per_tok, n_batched, __fma_rn(m.ctx_ms_per_tok, n_ctx, m.fixed_ms));
}

// One CTA.  Each thread accumulates, for every candidate k, the fixed-point token sum
// L(k) = sum_i rint(2^32 l(alpha_i, min(k, cap_i))) and sum_i min(k, cap_i); one warp
// reduction + one shared-memory step give the totals; lane k of warp 0 then evaluates
// T(k) and G(k) in parallel and lane 0 runs Listing 2's strict-'>' scan over k.
__global__ void __launch_bounds__(kGpThreads)
    goodput_choose_k_kernel(const double* __restrict__ alpha, int32_t alpha_per_request,
                            const int32_t* __restrict__ ctx_len, const int32_t* __restrict__ cap,
                            int32_t B, int32_t k_max, int32_t policy, tsv_latency_model target,
                            tsv_latency_model draft, double pld_cost_ms, long long kv_free,
                            int32_t* __restrict__ k_out, double* __restrict__ goodput_out,
                            int32_t* __restrict__ k_per_request) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ long long sL[kGpWarps][kGpMaxK];
    __shared__ long long sN[kGpWarps][kGpMaxK];
    __shared__ long long sC[kGpWarps][3];
    __shared__ int s_best;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long Lk[kGpMaxK], Nk[kGpMaxK];
#pragma unroll
    for (int k = 0; k < kGpMaxK; ++k) Lk[k] = Nk[k] = 0;
    long long n_ctx = 0, n_ctx_spec = 0, b_spec = 0;
    const double a_glob = alpha_per_request ? 0.0 : alpha[0];
    for (int32_t i = threadIdx.x; i < B; i += kGpThreads) {
        const double a = alpha_per_request ? alpha[i] : a_glob;
        const int32_t ci = cap[i];
        const int32_t cl = ctx_len[i];
        n_ctx += cl;
        if (ci > 0) {
            n_ctx_spec += cl;
            b_spec += 1;
        }
        double l = 1.0;  // l(a, 0); Horner step l(a, j+1) = fma(a, l(a, j), 1)
        long long fix = __double2ll_rn(l * 0x1p32);
        int32_t jcur = 0;
#pragma unroll
        for (int k = 0; k < kGpMaxK; ++k) {
            int32_t ki = k < ci ? k : ci;
            if (ki < 0) ki = 0;
            while (jcur < ki) {
                l = __fma_rn(a, l, 1.0);
                ++jcur;
                fix = __double2ll_rn(l * 0x1p32);
            }
            Lk[k] += fix;
            Nk[k] += ki;
        }
    }
#pragma unroll
    for (int k = 0; k < kGpMaxK; ++k) {
        if (k <= k_max) {
            const long long l = warp_sum_i64(Lk[k]);
            const long long n = warp_sum_i64(Nk[k]);
            if (lane == 0) {
                sL[warp][k] = l;
                sN[warp][k] = n;
            }
        }
    }
    n_ctx = warp_sum_i64(n_ctx);
    n_ctx_spec = warp_sum_i64(n_ctx_spec);
    b_spec = warp_sum_i64(b_spec);
    if (lane == 0) {
        sC[warp][0] = n_ctx;
        sC[warp][1] = n_ctx_spec;
        sC[warp][2] = b_spec;
    }
    __syncthreads();
    if (warp == 0) {
        long long c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
        for (int w = 0; w < kGpWarps; ++w) {
            c0 += sC[w][0];
            c1 += sC[w][1];
            c2 += sC[w][2];
        }
        double g = -1.0;
        bool valid = false;
        if (lane <= k_max) {
            long long L = 0, N = 0;
#pragma unroll
            for (int w = 0; w < kGpWarps; ++w) {
                L += sL[w][lane];
                N += sN[w][lane];
            }
            const long long n_batched = N + static_cast<long long>(B);
            if (!(lane > 0 && kv_free >= 0 && n_batched > kv_free)) {  // Listing 2 line 5: OOM -> skip
                const double t_target = fwd_time(target, static_cast<double>(c0), static_cast<double>(n_batched));
                double t_draft;
                if (policy == TSV_POLICY_PLD)
                    t_draft = pld_cost_ms;
                else
                    t_draft = lane > 0 ? __dmul_rn(static_cast<double>(lane),
                                                   fwd_time(draft, static_cast<double>(c1), static_cast<double>(c2)))
                                       : 0.0;
                g = __ddiv_rn(__dmul_rn(static_cast<double>(L), 0x1p-32), __dadd_rn(t_target, t_draft));
                valid = true;
            }
            if (goodput_out) goodput_out[lane] = g;
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
        if (lane == 0) {
            *k_out = best_k;
            s_best = best_k;
        }
    }
    if (k_per_request) {
        __syncthreads();
        const int32_t kb = s_best;
        for (int32_t i = threadIdx.x; i < B; i += kGpThreads) {
            int32_t ki = kb < cap[i] ? kb : cap[i];
            k_per_request[i] = ki < 0 ? 0 : ki;
        }
    }
}

__global__ void __launch_bounds__(kGpThreads)
    update_acceptance_kernel(double* __restrict__ alpha, int32_t per_request,
                             const int32_t* __restrict__ num_accepted, const int32_t* __restrict__ row_offsets,
                             int32_t B, double decay, int32_t estimator) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ long long red[kGpWarps][2];
    long long sm = 0, stt = 0;
    for (int32_t i = threadIdx.x; i < B; i += kGpThreads) {
        const int32_t k = row_offsets[i + 1] - row_offsets[i] - 1;
        const int32_t m = num_accepted[i];
        if (m < 0) continue;
        const long long t = estimator == TSV_EST_PROPOSED ? k : (m + (m < k ? 1 : 0));
        if (per_request) {
            if (t > 0) {
                const double r = __ddiv_rn(static_cast<double>(m), static_cast<double>(t));
                alpha[i] = __fma_rn(decay, __dsub_rn(alpha[i], r), r);
            }
        } else {
            sm += m;
            stt += t;
        }
    }
    if (per_request) return;
    sm = warp_sum_i64(sm);
    stt = warp_sum_i64(stt);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        red[warp][0] = sm;
        red[warp][1] = stt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long a = 0, b = 0;
#pragma unroll
        for (int w = 0; w < kGpWarps; ++w) {
            a += red[w][0];
            b += red[w][1];
        }
        if (b > 0) {
            const double r = __ddiv_rn(static_cast<double>(a), static_cast<double>(b));
            alpha[0] = __fma_rn(decay, __dsub_rn(alpha[0], r), r);
        }
    }
}

}  // namespace tsv

using namespace tsv;

extern "C" tsv_status tsv_goodput_choose_k(const double* alpha, int32_t alpha_per_request,
                                           const int32_t* ctx_len, const int32_t* cap, int32_t B,
                                           int32_t k_max, int32_t policy, tsv_latency_model target,
                                           tsv_latency_model draft, double pld_cost_ms,
                                           int64_t kv_free_slots, int32_t* k_out, double* goodput_out,
                                           int32_t* k_per_request, void* stream) {
    TSV_REQUIRE(B >= 1, "tsv_goodput_choose_k: B must be >= 1 (got %d)", B);
    TSV_REQUIRE(k_max >= 0 && k_max <= TSV_MAX_K, "tsv_goodput_choose_k: k_max %d outside [0, %d]", k_max, TSV_MAX_K);
    TSV_REQUIRE(policy == TSV_POLICY_DRAFT || policy == TSV_POLICY_PLD, "tsv_goodput_choose_k: unknown policy %d", policy);
    TSV_REQUIRE(alpha && ctx_len && cap && k_out, "tsv_goodput_choose_k: a required array is NULL");
    TSV_TRY(check_device());
    TSV_CUDA(launch_pdl(goodput_choose_k_kernel, dim3(1), dim3(kGpThreads), 0, static_cast<cudaStream_t>(stream),
                        alpha, alpha_per_request, ctx_len, cap, B, k_max, policy, target, draft, pld_cost_ms,
                        static_cast<long long>(kv_free_slots), k_out, goodput_out, k_per_request),
             "goodput_choose_k_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_update_acceptance(double* alpha, int32_t per_request, const int32_t* num_accepted,
                                            const int32_t* row_offsets, int32_t B, double decay,
                                            int32_t estimator, void* stream) {
    TSV_REQUIRE(B >= 0, "tsv_update_acceptance: B < 0");
    TSV_REQUIRE(decay >= 0.0 && decay <= 1.0, "tsv_update_acceptance: decay %g outside [0, 1]", decay);
    TSV_REQUIRE(estimator == TSV_EST_TESTED || estimator == TSV_EST_PROPOSED, "tsv_update_acceptance: unknown estimator");
    if (B == 0) return TSV_OK;
    TSV_REQUIRE(alpha && num_accepted && row_offsets, "tsv_update_acceptance: a required array is NULL");
    TSV_TRY(check_device());
    TSV_CUDA(launch_pdl(update_acceptance_kernel, dim3(1), dim3(kGpThreads), 0, static_cast<cudaStream_t>(stream),
                        alpha, per_request, num_accepted, row_offsets, B, decay, estimator),
             "update_acceptance_kernel launch");
    return TSV_OK;
}
