// loop.cu -- closed-loop harness kernels (reading R26 in DESIGN.md 3).
//
// The paper evaluates TurboSpec's controller on real models (k adapts to load
// and to the acceptance rate).  To exercise the same feedback loop on the device without model
// weights, a decode step is closed with a synthetic target and a context append:
//   lookup -> choose-k -> tsv_sim_target -> verify (+ alpha update) -> tsv_context_append,
// all asynchronous on one stream, so many steps replay as one CUDA graph.
#include <algorithm>

#include "common.cuh"

namespace tsv {

constexpr int kSimThreads = 1024;

// One CTA: row_offsets = exclusive scan of (k_i + 1), drafts packed at row_offsets[i] - i,
// row_info[r] = (request << 4) | position for every used row.
__global__ void __launch_bounds__(kSimThreads) sim_offsets_kernel(const int32_t* __restrict__ proposals, int32_t K,
                                                                  const int32_t* __restrict__ k_req, int32_t B,
                                                                  int32_t* __restrict__ row_offsets,
                                                                  int32_t* __restrict__ drafts,
                                                                  int32_t* __restrict__ row_info) {
    __shared__ int32_t s_warp[kSimThreads / 32];
    __shared__ int32_t s_carry;
    pdl_wait();
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int32_t base = 0; base < B; base += kSimThreads) {
        const int32_t i = base + threadIdx.x;
        const int32_t k = i < B ? k_req[i] : 0;
        const int32_t c = i < B ? k + 1 : 0;
        int32_t incl = c;  // warp inclusive scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int32_t w = s_warp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t t = __shfl_up_sync(0xFFFFFFFFu, w, o);
                if (lane >= o) w += t;
            }
            s_warp[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        const int32_t r0 = s_carry + (warp ? s_warp[warp - 1] : 0) + incl - c;
        if (i < B) {
            row_offsets[i] = r0;
            for (int32_t j = 0; j < k; ++j) drafts[r0 - i + j] = proposals[static_cast<int64_t>(i) * K + j];
            for (int32_t j = 0; j <= k; ++j) row_info[r0 + j] = (i << 4) | j;
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry += s_warp[kSimThreads / 32 - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) row_offsets[B] = s_carry;
}

// Every used row: draft rows put alpha_true on the draft and (1 - alpha_true) / (V - 1)
// elsewhere, bonus rows are uniform.  float4 stores; columns [V, ld) are zero.
__global__ void __launch_bounds__(256) sim_rows_kernel(const int32_t* __restrict__ proposals, int32_t K,
                                                       const int32_t* __restrict__ k_req,
                                                       const float* __restrict__ alpha_true, int32_t V, int64_t ld,
                                                       int32_t rows_cap, const int32_t* __restrict__ row_offsets,
                                                       const int32_t* __restrict__ row_info, int32_t B,
                                                       float* __restrict__ p) {
    pdl_wait();
    pdl_launch_dependents();
    const int32_t rows = min(rows_cap, row_offsets[B]);
    const float a = *alpha_true;
    const float rest = V > 1 ? __double2float_rn((1.0 - static_cast<double>(a)) / static_cast<double>(V - 1)) : 0.0f;
    const float unif = __double2float_rn(1.0 / static_cast<double>(V));
    const int64_t q4 = ld >> 2;
    const int64_t n = static_cast<int64_t>(rows) * q4;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t r = static_cast<int32_t>(e / q4);
        const int32_t f = static_cast<int32_t>(e % q4);
        const int32_t info = row_info[r];
        const int32_t i = info >> 4, j = info & 15;
        const bool draft_row = j < k_req[i];
        const int32_t x = draft_row ? proposals[static_cast<int64_t>(i) * K + j] : -1;
        const float base = draft_row ? rest : unif;
        float v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int32_t col = 4 * f + t;
            v[t] = col >= V ? 0.0f : (col == x ? a : base);
        }
        reinterpret_cast<float4*>(p + static_cast<int64_t>(r) * ld)[f] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// One CTA per request: out window = in[e..L) followed by the e = m_i + 1 emitted tokens.
__global__ void __launch_bounds__(256) context_append_kernel(const int32_t* __restrict__ ctx_in, int32_t L,
                                                             const int32_t* __restrict__ out_tokens,
                                                             const int32_t* __restrict__ num_accepted, int32_t k_max,
                                                             int32_t* __restrict__ ctx_out, int32_t* ctx_len) {
    pdl_wait();
    pdl_launch_dependents();
    const int32_t i = blockIdx.x;
    const int32_t m = num_accepted[i];
    int32_t e = m >= 0 ? m + 1 : 0;
    if (e > L) e = L;
    const int32_t* in = ctx_in + static_cast<int64_t>(i) * L;
    int32_t* out = ctx_out + static_cast<int64_t>(i) * L;
    const int32_t* em = out_tokens + static_cast<int64_t>(i) * (k_max + 1) + (m + 1 - e);
    for (int32_t t = threadIdx.x; t < L; t += blockDim.x) out[t] = t < L - e ? in[t + e] : em[t - (L - e)];
    if (threadIdx.x == 0 && m >= 0) ctx_len[i] += m + 1;
}

}  // namespace tsv

using namespace tsv;

extern "C" tsv_status tsv_sim_target(const int32_t* proposals, int32_t K, const int32_t* k_req, int32_t B,
                                     const float* alpha_true, int32_t V, int64_t ld, int32_t rows_cap, float* p_out,
                                     int32_t* row_offsets, int32_t* drafts, int32_t* row_info, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(B >= 0 && K >= 1 && K <= TSV_MAX_K, "tsv_sim_target: need B >= 0 and 1 <= K <= %d", TSV_MAX_K);
    TSV_REQUIRE(V >= 1 && ld >= V && ld % 4 == 0, "tsv_sim_target: need 1 <= V <= ld, ld %% 4 == 0");
    TSV_REQUIRE(rows_cap >= B * (K + 1), "tsv_sim_target: rows_cap %d < B (K + 1)", rows_cap);
    if (B == 0) return TSV_OK;
    TSV_REQUIRE(proposals && k_req && alpha_true && p_out && row_offsets && drafts && row_info,
                "tsv_sim_target: a required array is NULL");
    TSV_TRY(check_device());
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    TSV_CUDA(launch_pdl(sim_offsets_kernel, dim3(1), dim3(kSimThreads), 0, st, proposals, K, k_req, B, row_offsets,
                        drafts, row_info),
             "sim_offsets_kernel launch");
    const int64_t n = static_cast<int64_t>(rows_cap) * (ld >> 2);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
    TSV_CUDA(launch_pdl(sim_rows_kernel, dim3(static_cast<unsigned>(grid)), dim3(256), 0, st, proposals, K, k_req,
                        alpha_true, V, ld, rows_cap, static_cast<const int32_t*>(row_offsets),
                        static_cast<const int32_t*>(row_info), B, p_out),
             "sim_rows_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_context_append(const int32_t* ctx_in, int32_t L, int32_t B, const int32_t* out_tokens,
                                         const int32_t* num_accepted, int32_t k_max, int32_t* ctx_out,
                                         int32_t* ctx_len, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(B >= 0 && L >= 1 && k_max >= 0 && k_max <= TSV_MAX_K, "tsv_context_append: bad sizes");
    if (B == 0) return TSV_OK;
    TSV_REQUIRE(ctx_in && out_tokens && num_accepted && ctx_out && ctx_len && ctx_in != ctx_out,
                "tsv_context_append: NULL or aliased arrays");
    TSV_TRY(check_device());
    TSV_CUDA(launch_pdl(context_append_kernel, dim3(static_cast<unsigned>(B)), dim3(256), 0,
                        static_cast<cudaStream_t>(stream), ctx_in, L, out_tokens, num_accepted, k_max, ctx_out, ctx_len),
             "context_append_kernel launch");
    return TSV_OK;
}
