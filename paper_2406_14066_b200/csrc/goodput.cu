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
#include <algorithm>
#include <cmath>
#include <vector>

#include "goodput.cuh"

namespace tsv {

#ifndef TSV_GP_CHOOSE_THREADS
#define TSV_GP_CHOOSE_THREADS 256
#endif
constexpr int kGpChooseThreads = TSV_GP_CHOOSE_THREADS;  // B = 256 step: 256 threads 2.84 us; 128: 3.12; 64: 3.86; 32: 6.10
// Before the grid-dependency wait: prefetch the context lengths (a step input that may have left L2 since
// it was last read) and alpha into L2, so the loads after the wait are L2 hits.  A prefetch returns no
// data and L2 is the coherence point for writes, so this is safe whatever is still in flight.
#ifndef TSV_GP_PREFETCH
#define TSV_GP_PREFETCH 1
#endif
__device__ __forceinline__ void gp_prefetch(const ChooseArgs& A) {
    if (!TSV_GP_PREFETCH) return;
    const int32_t line = static_cast<int32_t>(threadIdx.x) * 32;  // one 128-byte line of ctx_len per thread
    if (line < A.B) prefetch_l2(A.ctx_len + line);
    if (threadIdx.x == 0) prefetch_l2(A.alpha);
}

__global__ void __launch_bounds__(kGpChooseThreads) goodput_choose_k_kernel(const ChooseArgs A) {
    TSV_STEP_SPAN(1);
    gp_prefetch(A);
    pdl_wait();
    TSV_STEP_WAITED();
    pdl_launch_dependents();
#if TSV_STEP_TRACE
    {  // choose_k_block with marks: m1 after the batch sums, m2 after Listing 2's argmax
        __shared__ int s_best;
        int32_t caps[kGpCapCache];
        const GpTotals t = gp_sums_block<kGpChooseThreads>(A, caps);
        TSV_STEP_MARK(1);
        if ((threadIdx.x >> 5) == 0) {
            const int kb = gp_argmax_warp(A, t);
            if (threadIdx.x == 0) s_best = kb;
        }
        TSV_STEP_MARK(2);
        if (A.k_per_request) {
            __syncthreads();
            gp_write_k_per_request<kGpChooseThreads>(A, s_best, caps);
        }
    }
#else
    choose_k_block<kGpChooseThreads>(A);
#endif
}

// Request-sharded ArgMaxGoodput in ONE kernel (the exchange step fused with its
// producer and consumer): this rank's exact int64 batch sums, summed over the ranks through
// NVLink peer memory (p2p.cuh), then Listing 2 on the global sums -- bit-identical to one device
// holding the whole batch.  k_i = min(k*, cap_i) for this rank's requests.
__global__ void __launch_bounds__(kGpChooseThreads) goodput_choose_k_p2p_kernel(const ChooseArgs A, const P2PView V,
                                                                              int32_t* devstatus) {
    __shared__ long long s_sums[2 * kGpMaxK + 4];
    __shared__ int s_best;
    gp_prefetch(A);
    pdl_wait();
    pdl_launch_dependents();
    int32_t caps[kGpCapCache];
    const GpTotals t = gp_sums_block<kGpChooseThreads>(A, caps);
    const int lane = threadIdx.x & 31;
    const int32_t K1 = A.k_max + 1;
    if (threadIdx.x < 32) {
        if (lane <= A.k_max) {
            s_sums[lane] = t.L;
            s_sums[K1 + lane] = t.N;
        }
        if (lane == 0) {
            s_sums[2 * K1] = t.c0;
            s_sums[2 * K1 + 1] = t.c1;
            s_sums[2 * K1 + 2] = t.c2;
            s_sums[2 * K1 + 3] = t.c3;
        }
    }
    __syncthreads();
    p2p_allreduce_block(s_sums, 2 * K1 + 4, V, devstatus);  // ends with a CTA barrier
    if (threadIdx.x < 32) {
        GpTotals g;
        g.L = lane <= A.k_max ? s_sums[lane] : 0;
        g.N = lane <= A.k_max ? s_sums[K1 + lane] : 0;
        g.c0 = s_sums[2 * K1];
        g.c1 = s_sums[2 * K1 + 1];
        g.c2 = s_sums[2 * K1 + 2];
        g.c3 = s_sums[2 * K1 + 3];
        const int kb = gp_argmax_warp(A, g);
        if (lane == 0) s_best = kb;
    }
    if (A.k_per_request && A.B > 0) {
        __syncthreads();
        gp_write_k_per_request<kGpChooseThreads>(A, s_best, caps);
    }
}

__global__ void __launch_bounds__(kGpThreads) update_acceptance_kernel(const UpdateArgs A) {
    pdl_wait();
    pdl_launch_dependents();
    update_block(A);
}

// Request-sharded mode: the batch sums of this rank's requests ...
__global__ void __launch_bounds__(kGpThreads) goodput_partial_kernel(const ChooseArgs A, long long* sums) {
    pdl_wait();
    pdl_launch_dependents();
    const GpTotals t = gp_sums_block(A);
    const int lane = threadIdx.x & 31;
    if ((threadIdx.x >> 5) == 0) {
        if (lane <= A.k_max) {
            sums[lane] = t.L;
            sums[A.k_max + 1 + lane] = t.N;
        }
        if (lane == 0) {
            long long* c = sums + 2 * (A.k_max + 1);
            c[0] = t.c0;
            c[1] = t.c1;
            c[2] = t.c2;
            c[3] = t.c3;
        }
    }
}

// ... and, after the element-wise sum over ranks, the argmax on the global sums.
__global__ void __launch_bounds__(kGpThreads) goodput_finalize_kernel(const ChooseArgs A, const long long* sums) {
    __shared__ int s_best;
    pdl_wait();
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31;
    if ((threadIdx.x >> 5) == 0) {
        const long long* c = sums + 2 * (A.k_max + 1);
        GpTotals t;
        t.L = lane <= A.k_max ? sums[lane] : 0;
        t.N = lane <= A.k_max ? sums[A.k_max + 1 + lane] : 0;
        t.c0 = c[0];
        t.c1 = c[1];
        t.c2 = c[2];
        t.c3 = c[3];
        const int kb = gp_argmax_warp(A, t);
        if (lane == 0) s_best = kb;
    }
    if (A.k_per_request && A.cap && A.B > 0) {
        __syncthreads();
        gp_write_k_per_request(A, s_best);
    }
}

__global__ void __launch_bounds__(kGpThreads) update_partial_kernel(const UpdateArgs A, long long* sums) {
    pdl_wait();
    pdl_launch_dependents();
    update_block(A, sums);
}

__global__ void update_finalize_kernel(double* alpha, const long long* sums, double decay) {
    pdl_wait();
    pdl_launch_dependents();
    if (threadIdx.x == 0) ewma_apply(alpha, sums[0], sums[1], decay);
}

// Batched ArgMaxGoodput (config 5 sweeps): one CTA per independent instance n, which owns
// requests [inst_offsets[n], inst_offsets[n+1]) of the concatenated ctx_len / cap arrays and
// the global alpha[n]; identical arithmetic to tsv_goodput_choose_k per instance.
#ifndef TSV_GP_BATCH_THREADS
#define TSV_GP_BATCH_THREADS 32
#endif
constexpr int kGpBatchThreads = TSV_GP_BATCH_THREADS;  // one warp per instance: all instances resident at once (config 5: 15.8 us; 64: 16.5; 128: 20.7; 256: 31.1)
__global__ void __launch_bounds__(kGpBatchThreads) goodput_choose_k_batched_kernel(ChooseArgs A, const int32_t* inst_offsets,
                                                                            int32_t n_inst) {
    pdl_wait();
    pdl_launch_dependents();
    const int32_t n = blockIdx.x;
    if (n >= n_inst) return;
    const int32_t lo = inst_offsets[n], hi = inst_offsets[n + 1];
    ChooseArgs B = A;
    B.alpha = A.alpha + n;
    B.alpha_per_request = 0;
    B.ctx_len = A.ctx_len + lo;
    B.cap = A.cap + lo;
    B.B = hi - lo;
    B.k_out = A.k_out + n;
    B.goodput_out = A.goodput_out ? A.goodput_out + static_cast<int64_t>(n) * (A.k_max + 1) : nullptr;
    B.k_per_request = A.k_per_request ? A.k_per_request + lo : nullptr;
    choose_k_block<kGpBatchThreads>(B);
}

}  // namespace tsv

using namespace tsv;
TSV_STEP_TRACE_READER(goodput)

extern "C" tsv_status tsv_goodput_choose_k_batched(const double* alpha, const int32_t* ctx_len, const int32_t* cap,
                                                   const int32_t* inst_offsets, int32_t n_inst, int32_t k_max,
                                                   int32_t policy, tsv_latency_model target, tsv_latency_model draft,
                                                   double pld_cost_ms, int64_t kv_free_slots, int32_t* k_out,
                                                   double* goodput_out, int32_t* k_per_request, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(n_inst >= 0, "tsv_goodput_choose_k_batched: n_inst < 0");
    TSV_REQUIRE(k_max >= 0 && k_max <= TSV_MAX_K, "tsv_goodput_choose_k_batched: k_max %d outside [0, %d]", k_max, TSV_MAX_K);
    TSV_REQUIRE(policy == TSV_POLICY_DRAFT || policy == TSV_POLICY_PLD, "tsv_goodput_choose_k_batched: unknown policy");
    if (n_inst == 0) return TSV_OK;
    TSV_REQUIRE(alpha && ctx_len && cap && inst_offsets && k_out, "tsv_goodput_choose_k_batched: a required array is NULL");
    TSV_TRY(check_device());
    ChooseArgs A = {};
    A.alpha = alpha;
    A.ctx_len = ctx_len;
    A.cap = cap;
    A.k_out = k_out;
    A.goodput_out = goodput_out;
    A.k_per_request = k_per_request;
    A.target = target;
    A.draft = draft;
    A.pld_cost_ms = pld_cost_ms;
    A.kv_free = static_cast<long long>(kv_free_slots);
    A.k_max = k_max;
    A.policy = policy;
    TSV_CUDA(launch_pdl(goodput_choose_k_batched_kernel, dim3(static_cast<unsigned>(n_inst)), dim3(kGpBatchThreads), 0,
                        static_cast<cudaStream_t>(stream), A, inst_offsets, n_inst),
             "goodput_choose_k_batched_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_goodput_partial(const double* alpha, int32_t alpha_per_request, const int32_t* ctx_len,
                                          const int32_t* cap, int32_t B, int32_t k_max, int64_t* sums,
                                          void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(B >= 0, "tsv_goodput_partial: B < 0 (%d)", B);
    TSV_REQUIRE(k_max >= 0 && k_max <= TSV_MAX_K, "tsv_goodput_partial: k_max %d outside [0, %d]", k_max, TSV_MAX_K);
    TSV_REQUIRE(sums != nullptr, "tsv_goodput_partial: sums is NULL");
    TSV_REQUIRE(B == 0 || (alpha && ctx_len && cap), "tsv_goodput_partial: a required array is NULL");
    TSV_TRY(check_device());
    ChooseArgs A = {};
    A.alpha = alpha;
    A.ctx_len = ctx_len;
    A.cap = cap;
    A.alpha_per_request = alpha_per_request;
    A.B = B;
    A.k_max = k_max;
    if (B == 0) {  // an empty request set: all sums are zero (alpha is not read)
        TSV_CUDA(cudaMemsetAsync(sums, 0, sizeof(int64_t) * TSV_GP_SUMS(k_max), static_cast<cudaStream_t>(stream)),
                 "cudaMemsetAsync");
        return TSV_OK;
    }
    TSV_CUDA(launch_pdl(goodput_partial_kernel, dim3(1), dim3(kGpThreads), 0, static_cast<cudaStream_t>(stream), A,
                        reinterpret_cast<long long*>(sums)),
             "goodput_partial_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_goodput_finalize(const int64_t* sums, int32_t k_max, int32_t policy,
                                           tsv_latency_model target, tsv_latency_model draft, double pld_cost_ms,
                                           int64_t kv_free_slots, const int32_t* cap, int32_t B_local,
                                           int32_t* k_out, double* goodput_out, int32_t* k_per_request,
                                           void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(k_max >= 0 && k_max <= TSV_MAX_K, "tsv_goodput_finalize: k_max %d outside [0, %d]", k_max, TSV_MAX_K);
    TSV_REQUIRE(policy == TSV_POLICY_DRAFT || policy == TSV_POLICY_PLD, "tsv_goodput_finalize: unknown policy %d", policy);
    TSV_REQUIRE(sums && k_out, "tsv_goodput_finalize: a required array is NULL");
    TSV_REQUIRE(B_local >= 0, "tsv_goodput_finalize: B_local < 0");
    TSV_REQUIRE(!k_per_request || B_local == 0 || cap, "tsv_goodput_finalize: k_per_request needs cap");
    TSV_TRY(check_device());
    ChooseArgs A = {};
    A.cap = cap;
    A.k_out = k_out;
    A.goodput_out = goodput_out;
    A.k_per_request = k_per_request;
    A.target = target;
    A.draft = draft;
    A.pld_cost_ms = pld_cost_ms;
    A.kv_free = static_cast<long long>(kv_free_slots);
    A.B = B_local;
    A.k_max = k_max;
    A.policy = policy;
    TSV_CUDA(launch_pdl(goodput_finalize_kernel, dim3(1), dim3(kGpThreads), 0, static_cast<cudaStream_t>(stream), A,
                        reinterpret_cast<const long long*>(sums)),
             "goodput_finalize_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_update_partial(const int32_t* num_accepted, const int32_t* row_offsets, int32_t B,
                                         int32_t estimator, int64_t* sums, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(B >= 0, "tsv_update_partial: B < 0");
    TSV_REQUIRE(estimator == TSV_EST_TESTED || estimator == TSV_EST_PROPOSED, "tsv_update_partial: unknown estimator");
    TSV_REQUIRE(sums != nullptr, "tsv_update_partial: sums is NULL");
    TSV_REQUIRE(B == 0 || (num_accepted && row_offsets), "tsv_update_partial: a required array is NULL");
    TSV_TRY(check_device());
    if (B == 0) {
        TSV_CUDA(cudaMemsetAsync(sums, 0, 2 * sizeof(int64_t), static_cast<cudaStream_t>(stream)), "cudaMemsetAsync");
        return TSV_OK;
    }
    UpdateArgs A = {};
    A.num_accepted = num_accepted;
    A.row_offsets = row_offsets;
    A.B = B;
    A.estimator = estimator;
    TSV_CUDA(launch_pdl(update_partial_kernel, dim3(1), dim3(kGpThreads), 0, static_cast<cudaStream_t>(stream), A,
                        reinterpret_cast<long long*>(sums)),
             "update_partial_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_update_finalize(double* alpha, const int64_t* sums, double decay, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(alpha && sums, "tsv_update_finalize: NULL argument");
    TSV_REQUIRE(decay >= 0.0 && decay <= 1.0, "tsv_update_finalize: decay %g outside [0, 1]", decay);
    TSV_TRY(check_device());
    TSV_CUDA(launch_pdl(update_finalize_kernel, dim3(1), dim3(32), 0, static_cast<cudaStream_t>(stream), alpha,
                        reinterpret_cast<const long long*>(sums), decay),
             "update_finalize_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_goodput_choose_k(const double* alpha, int32_t alpha_per_request,
                                           const int32_t* ctx_len, const int32_t* cap, int32_t B,
                                           int32_t k_max, int32_t policy, tsv_latency_model target,
                                           tsv_latency_model draft, double pld_cost_ms,
                                           int64_t kv_free_slots, int32_t* k_out, double* goodput_out,
                                           int32_t* k_per_request, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(B >= 1, "tsv_goodput_choose_k: B must be >= 1 (got %d)", B);
    TSV_REQUIRE(k_max >= 0 && k_max <= TSV_MAX_K, "tsv_goodput_choose_k: k_max %d outside [0, %d]", k_max, TSV_MAX_K);
    TSV_REQUIRE(policy == TSV_POLICY_DRAFT || policy == TSV_POLICY_PLD, "tsv_goodput_choose_k: unknown policy %d", policy);
    TSV_REQUIRE(alpha && ctx_len && cap && k_out, "tsv_goodput_choose_k: a required array is NULL");
    TSV_TRY(check_device());
    ChooseArgs A;
    A.alpha = alpha;
    A.ctx_len = ctx_len;
    A.cap = cap;
    A.k_out = k_out;
    A.goodput_out = goodput_out;
    A.k_per_request = k_per_request;
    A.target = target;
    A.draft = draft;
    A.pld_cost_ms = pld_cost_ms;
    A.kv_free = static_cast<long long>(kv_free_slots);
    A.alpha_per_request = alpha_per_request;
    A.B = B;
    A.k_max = k_max;
    A.policy = policy;
    TSV_CUDA(launch_pdl(goodput_choose_k_kernel, dim3(1), dim3(kGpChooseThreads), 0, static_cast<cudaStream_t>(stream), A),
             "goodput_choose_k_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_update_acceptance(double* alpha, int32_t per_request, const int32_t* num_accepted,
                                            const int32_t* row_offsets, int32_t B, double decay,
                                            int32_t estimator, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(B >= 0, "tsv_update_acceptance: B < 0");
    TSV_REQUIRE(decay >= 0.0 && decay <= 1.0, "tsv_update_acceptance: decay %g outside [0, 1]", decay);
    TSV_REQUIRE(estimator == TSV_EST_TESTED || estimator == TSV_EST_PROPOSED, "tsv_update_acceptance: unknown estimator");
    if (B == 0) return TSV_OK;
    TSV_REQUIRE(alpha && num_accepted && row_offsets, "tsv_update_acceptance: a required array is NULL");
    TSV_TRY(check_device());
    UpdateArgs A = {};
    A.alpha = alpha;
    A.num_accepted = num_accepted;
    A.row_offsets = row_offsets;
    A.decay = decay;
    A.per_request = per_request;
    A.B = B;
    A.estimator = estimator;
    TSV_CUDA(launch_pdl(update_acceptance_kernel, dim3(1), dim3(kGpThreads), 0, static_cast<cudaStream_t>(stream), A),
             "update_acceptance_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_goodput_choose_k_p2p(const double* alpha, int32_t alpha_per_request, const int32_t* ctx_len,
                                               const int32_t* cap, int32_t B, int32_t k_max, int32_t policy,
                                               tsv_latency_model target, tsv_latency_model draft, double pld_cost_ms,
                                               int64_t kv_free_slots, int32_t* k_out, double* goodput_out,
                                               int32_t* k_per_request, tsv_p2p* p, int32_t* device_status,
                                               void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(B >= 0, "tsv_goodput_choose_k_p2p: B < 0 (%d)", B);
    TSV_REQUIRE(k_max >= 0 && k_max <= TSV_MAX_K, "tsv_goodput_choose_k_p2p: k_max %d outside [0, %d]", k_max, TSV_MAX_K);
    TSV_REQUIRE(policy == TSV_POLICY_DRAFT || policy == TSV_POLICY_PLD, "tsv_goodput_choose_k_p2p: unknown policy %d",
                policy);
    TSV_REQUIRE(p != nullptr, "tsv_goodput_choose_k_p2p: p2p handle is NULL");
    TSV_REQUIRE(alpha && k_out && (B == 0 || (ctx_len && cap)), "tsv_goodput_choose_k_p2p: a required array is NULL");
    TSV_TRY(check_device());
    ChooseArgs A = {};
    A.alpha = alpha;
    A.ctx_len = ctx_len;
    A.cap = cap;
    A.k_out = k_out;
    A.goodput_out = goodput_out;
    A.k_per_request = k_per_request;
    A.target = target;
    A.draft = draft;
    A.pld_cost_ms = pld_cost_ms;
    A.kv_free = static_cast<long long>(kv_free_slots);
    A.alpha_per_request = alpha_per_request;
    A.B = B;
    A.k_max = k_max;
    A.policy = policy;
    TSV_CUDA(launch_pdl(goodput_choose_k_p2p_kernel, dim3(1), dim3(kGpChooseThreads), 0,
                        static_cast<cudaStream_t>(stream), A, p->view, device_status),
             "goodput_choose_k_p2p_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_update_acceptance_p2p(double* alpha, int32_t per_request, const int32_t* num_accepted,
                                                const int32_t* row_offsets, int32_t B, double decay, int32_t estimator,
                                                tsv_p2p* p, int32_t* device_status, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(B >= 0, "tsv_update_acceptance_p2p: B < 0");
    TSV_REQUIRE(decay >= 0.0 && decay <= 1.0, "tsv_update_acceptance_p2p: decay %g outside [0, 1]", decay);
    TSV_REQUIRE(estimator == TSV_EST_TESTED || estimator == TSV_EST_PROPOSED,
                "tsv_update_acceptance_p2p: unknown estimator");
    TSV_REQUIRE(p != nullptr && alpha != nullptr, "tsv_update_acceptance_p2p: NULL argument");
    TSV_REQUIRE(B == 0 || (num_accepted && row_offsets), "tsv_update_acceptance_p2p: a required array is NULL");
    if (per_request && B == 0) return TSV_OK;  // per-request alphas: no exchange
    TSV_TRY(check_device());
    UpdateArgs A = {};
    A.alpha = alpha;
    A.num_accepted = num_accepted;
    A.row_offsets = row_offsets;
    A.decay = decay;
    A.per_request = per_request;
    A.B = B;
    A.estimator = estimator;
    A.use_p2p = per_request ? 0 : 1;
    A.devstatus = device_status;
    A.p2p = p->view;
    TSV_CUDA(launch_pdl(update_acceptance_kernel, dim3(1), dim3(kGpThreads), 0, static_cast<cudaStream_t>(stream), A),
             "update_acceptance_kernel launch");
    return TSV_OK;
}

// ---------------------------------------------------------------- latency-model fit (host)
// Reading R25: OLS of the measured forward time on
// (N_context, N_batched, 1), clamp-and-refit of negative coefficients, R^2.  Host code (a
// profiling-time fit of a handful of samples); least squares by Householder QR of the
// column-scaled design, so no normal equations are formed.
namespace {
// min ||X b - y|| over the columns in `cols` (X column-major n x 3); false if rank-deficient.
bool qr_lstsq(const std::vector<double>& X, const std::vector<double>& y, int n, const int* cols, int m,
              double beta[3]) {
    std::vector<double> A(static_cast<size_t>(n) * m), r(y);
    double scale[3];
    for (int j = 0; j < m; ++j) {
        double nrm = 0.0;
        for (int i = 0; i < n; ++i) nrm = std::max(nrm, std::fabs(X[static_cast<size_t>(cols[j]) * n + i]));
        scale[j] = nrm > 0.0 ? nrm : 1.0;
        for (int i = 0; i < n; ++i) A[static_cast<size_t>(j) * n + i] = X[static_cast<size_t>(cols[j]) * n + i] / scale[j];
    }
    double R[3][3] = {};
    for (int j = 0; j < m; ++j) {
        double* a = &A[static_cast<size_t>(j) * n];
        double nrm = 0.0;
        for (int i = j; i < n; ++i) nrm += a[i] * a[i];
        nrm = std::sqrt(nrm);
        if (!(nrm > 1e-10 * std::sqrt(static_cast<double>(n)))) return false;  // dependent column
        const double alpha = a[j] > 0 ? -nrm : nrm;
        std::vector<double> v(a + j, a + n);
        v[0] -= alpha;
        double vv = 0.0;
        for (double t : v) vv += t * t;
        auto reflect = [&](double* col) {
            double d = 0.0;
            for (int i = j; i < n; ++i) d += v[i - j] * col[i];
            const double f = 2.0 * d / vv;
            for (int i = j; i < n; ++i) col[i] -= f * v[i - j];
        };
        if (vv > 0.0) {
            for (int k = j; k < m; ++k) reflect(&A[static_cast<size_t>(k) * n]);
            reflect(r.data());
        }
        for (int k = j; k < m; ++k) R[j][k] = A[static_cast<size_t>(k) * n + j];
    }
    double z[3] = {};
    for (int j = m - 1; j >= 0; --j) {
        double t = r[j];
        for (int k = j + 1; k < m; ++k) t -= R[j][k] * z[k];
        z[j] = t / R[j][j];
    }
    for (int i = 0; i < 3; ++i) beta[i] = 0.0;
    for (int j = 0; j < m; ++j) beta[cols[j]] = z[j] / scale[j];
    return true;
}
}  // namespace

extern "C" tsv_status tsv_fit_latency_model(const double* ctx_tokens, const double* batched_tokens,
                                            const double* ms, int32_t n, tsv_latency_model* out, double* r2_out) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(n >= 3, "tsv_fit_latency_model: TooFewSamples (n = %d < 3)", n);
    TSV_REQUIRE(ctx_tokens && batched_tokens && ms && out, "tsv_fit_latency_model: NULL argument");
    std::vector<double> X(3 * static_cast<size_t>(n)), y(ms, ms + n);
    for (int32_t i = 0; i < n; ++i) {
        X[i] = ctx_tokens[i];
        X[static_cast<size_t>(n) + i] = batched_tokens[i];
        X[2 * static_cast<size_t>(n) + i] = 1.0;
    }
    double beta[3];
    int cols[3] = {0, 1, 2};
    TSV_REQUIRE(qr_lstsq(X, y, n, cols, 3, beta), "tsv_fit_latency_model: DegenerateDesign (collinear regressors)");
    bool free_[3] = {true, true, true};
    for (;;) {  // clamp every negative free coefficient, refit the rest
        bool neg = false;
        for (int i = 0; i < 3; ++i)
            if (free_[i] && beta[i] < 0.0) {
                free_[i] = false;
                neg = true;
            }
        if (!neg) break;
        int m = 0;
        for (int i = 0; i < 3; ++i)
            if (free_[i]) cols[m++] = i;
        if (m == 0) {
            beta[0] = beta[1] = beta[2] = 0.0;
            break;
        }
        if (!qr_lstsq(X, y, n, cols, m, beta)) break;
    }
    double mean = 0.0, ss_res = 0.0, ss_tot = 0.0;
    for (int32_t i = 0; i < n; ++i) mean += ms[i];
    mean /= n;
    for (int32_t i = 0; i < n; ++i) {
        const double pred = beta[0] * ctx_tokens[i] + beta[1] * batched_tokens[i] + beta[2];
        ss_res += (ms[i] - pred) * (ms[i] - pred);
        ss_tot += (ms[i] - mean) * (ms[i] - mean);
    }
    out->ctx_ms_per_tok = beta[0];
    out->batched_ms_per_tok = beta[1];
    out->fixed_ms = beta[2];
    if (r2_out) *r2_out = ss_tot > 0.0 ? 1.0 - ss_res / ss_tot : (ss_res == 0.0 ? 1.0 : 0.0);
    return TSV_OK;
}
