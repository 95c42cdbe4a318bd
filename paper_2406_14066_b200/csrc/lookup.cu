// lookup.cu -- prompt-lookup n-gram proposal (PLD) on sm_100a (K2).
// PAPER.md:57 [AD] (fixed-length proposal; cost depends only on the context search),
// PAPER.md:454, 498 (n-grams retrieved from the prompt), Fig. PAPER.md:44-49
// (a request with no match proposes nothing); reading R20 in DESIGN.md section 3.
//
// "Longest n in [n_min, n_max] with a match, then the latest start" is evaluated as
// ONE max-reduction: for every end position e in [0, L-2] let c(e)
// be the length of the common suffix of ctx[..e] and ctx[..L-1] capped at n_max;
// key(e) = (c(e) << 20) | e.  The lexicographic max of (c, e) is exactly the longest
// matching n and, among its matches, the latest one.
//
// One CTA per request reads the context straight from global memory in 16-byte groups
// aligned to the ctx allocation (no staging, no barrier wait): thread t takes groups
// g_lo+t, g_lo+t+256, ..., loading kUnroll groups before it compares any.  For the four
// positions of a group it also needs the three tokens before them (the previous group,
// an L1 hit: the neighbouring thread loads it too).  The first min(n_max, 4) suffix
// comparisons are evaluated branch-free on that 7-token window; only a position whose
// 4-token suffix already matches and n_max > 4 walks further (rarely).  A block max
// reduction (redux.sync + shared memory) gives the request's key; warp 0 writes the
// proposal.
#include "goodput.cuh"

namespace tsv {

#ifndef TSV_LOOKUP_THREADS
#define TSV_LOOKUP_THREADS 1024
#endif
#ifndef TSV_LOOKUP_UNROLL
#define TSV_LOOKUP_UNROLL 1
#endif
constexpr int kLookupThreads = TSV_LOOKUP_THREADS;  // the fused variant's tail is written for any multiple of 32

// Fused lookup + choose-k scratch (TSV_LOOKUP_CHOOSE_SCRATCH bytes, zero when idle): the batch sums
// of ArgMaxGoodput accumulated by every CTA with integer atomics, and the arrival counter.
struct FusedScratch {
    unsigned int counter;
    unsigned int pad;
    unsigned long long L[kGpMaxK];  // sum_i rint(2^32 l(alpha_i, min(k, cap_i)))  (two's complement add)
    unsigned long long N[kGpMaxK];  // sum_i min(k, cap_i)
    unsigned long long C[3];        // sum ctx_len, sum ctx_len over cap > 0, #{cap > 0}
};
static_assert(sizeof(FusedScratch) <= TSV_LOOKUP_CHOOSE_SCRATCH, "scratch size");
constexpr int kLookupUnroll = TSV_LOOKUP_UNROLL;  // groups in flight per thread

struct Group {
    int4 cur;   // ctx[4g .. 4g+3]
    int4 prev;  // ctx[4g-4 .. 4g-1] (only .y .z .w are used)
};

// Loads group g; `last` is the absolute index of the request's last token (every index
// read is <= last, so nothing past the request is touched; indices below the request's
// offset are valid memory and are masked by e - j >= 0 in scan_group).
__device__ __forceinline__ Group load_group(const int32_t* __restrict__ ctx, int64_t g, int64_t last, bool vec) {
    Group G;
    const int64_t a = 4 * g;
    if (vec && a + 3 <= last) {
        G.cur = __ldg(reinterpret_cast<const int4*>(ctx) + g);
    } else {
        G.cur.x = a <= last ? __ldg(ctx + a) : 0;
        G.cur.y = a + 1 <= last ? __ldg(ctx + a + 1) : 0;
        G.cur.z = a + 2 <= last ? __ldg(ctx + a + 2) : 0;
        G.cur.w = a + 3 <= last ? __ldg(ctx + a + 3) : 0;
    }
    if (g == 0) {
        G.prev = make_int4(0, 0, 0, 0);
    } else if (vec) {
        G.prev = __ldg(reinterpret_cast<const int4*>(ctx) + g - 1);
    } else {
        G.prev = make_int4(0, __ldg(ctx + a - 3), __ldg(ctx + a - 2), __ldg(ctx + a - 1));
    }
    return G;
}

struct Query {
    int32_t q0, q1, q2, q3;  // q_j = ctx[L-1-j] (0 where j >= L: masked by e - j >= 0)
    int32_t off, L, n_max;
};

// key(e) = (c(e) << 20) | e for the four positions of group g (0 when c(e) = 0 or e is
// not an end position in [0, L-2]); returns their max.
__device__ __forceinline__ uint32_t scan_group(const int32_t* __restrict__ ctx, const Group& G, int64_t g,
                                               const Query& Q) {
    const int32_t w[7] = {G.prev.y, G.prev.z, G.prev.w, G.cur.x, G.cur.y, G.cur.z, G.cur.w};
    uint32_t best = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int64_t e = 4 * g + s - Q.off;
        const bool m0 = e >= 0 && e <= Q.L - 2 && w[3 + s] == Q.q0;
        const bool m1 = m0 && Q.n_max >= 2 && e >= 1 && w[2 + s] == Q.q1;
        const bool m2 = m1 && Q.n_max >= 3 && e >= 2 && w[1 + s] == Q.q2;
        const bool m3 = m2 && Q.n_max >= 4 && e >= 3 && w[s] == Q.q3;
        int32_t cl = static_cast<int32_t>(m0) + static_cast<int32_t>(m1) + static_cast<int32_t>(m2) +
                     static_cast<int32_t>(m3);
        if (m3 && Q.n_max > 4) {  // rare: the 4-token suffix matches and longer n-grams count
            const int32_t* c = ctx + Q.off;
            const int32_t ee = static_cast<int32_t>(e);
            while (cl < Q.n_max && cl <= ee && __ldg(c + ee - cl) == __ldg(c + Q.L - 1 - cl)) ++cl;
        }
        const uint32_t key = cl ? ((static_cast<uint32_t>(cl) << 20) | static_cast<uint32_t>(e)) : 0u;
        best = key > best ? key : best;
    }
    return best;
}

// Fused ArgMaxGoodput (CTA-wide, after request i's proposal length is written): warp 0 adds
// request i's terms of the batch sums with integer atomics (exact, any order: the same sums
// as choose_k_block), then the CTA that arrives last evaluates G(k) from the sums, writes k*,
// the goodput values and k_i for every request, and re-zeroes the scratch.
__device__ __forceinline__ void fused_choose_k(const ChooseArgs& A, FusedScratch* S, int32_t i, int32_t ci) {
    __shared__ int s_last, s_best;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {  // ci: request i's proposal length (valid in warp 0)
        if (A.alpha_ready) wait_alpha_ready(A.alpha_ready, A.devstatus);  // alpha may be written by a kernel in flight
        const double a = __ldcg(A.alpha + (A.alpha_per_request ? i : 0));
        const int32_t k = lane;
        if (k <= A.k_max) {
            int32_t ki = k < ci ? k : ci;
            if (ki < 0) ki = 0;
            double l = 1.0;  // l(a, ki) by Horner, op-for-op choose_k_block
            for (int32_t j = 0; j < ki; ++j) l = __fma_rn(a, l, 1.0);
            atomicAdd(&S->L[k], static_cast<unsigned long long>(__double2ll_rn(l * 0x1p32)));
            atomicAdd(&S->N[k], static_cast<unsigned long long>(ki));
        }
        if (lane == 0) {
            const int32_t cl = __ldcg(A.ctx_len + i);
            atomicAdd(&S->C[0], static_cast<unsigned long long>(static_cast<long long>(cl)));
            if (ci > 0) {
                atomicAdd(&S->C[1], static_cast<unsigned long long>(static_cast<long long>(cl)));
                atomicAdd(&S->C[2], 1ull);
            }
        }
        __threadfence();  // this request's terms (and proposal row) before the arrival
        __syncwarp();
        if (lane == 0) {
            const unsigned int prev = atomicAdd(&S->counter, 1u);
            s_last = prev == static_cast<unsigned int>(A.B) - 1u;
        }
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < 32) {
        GpTotals t;
        t.L = lane <= A.k_max ? static_cast<long long>(atomicAdd(&S->L[lane], 0ull)) : 0;
        t.N = lane <= A.k_max ? static_cast<long long>(atomicAdd(&S->N[lane], 0ull)) : 0;
        t.c0 = static_cast<long long>(atomicAdd(&S->C[0], 0ull));
        t.c1 = static_cast<long long>(atomicAdd(&S->C[1], 0ull));
        t.c2 = static_cast<long long>(atomicAdd(&S->C[2], 0ull));
        t.c3 = A.B;
        const int kb = gp_argmax_warp(A, t);
        if (lane == 0) s_best = kb;
        if (lane < kGpMaxK) {  // idle again for the next call
            S->L[lane] = 0ull;
            S->N[lane] = 0ull;
        }
        if (lane < 3) S->C[lane] = 0ull;
        if (lane == 0) S->counter = 0u;
    }
    if (A.k_per_request) {
        __syncthreads();
        gp_write_k_per_request(A, s_best);
    }
}

// FUSED: the CTA that finishes last also runs ArgMaxGoodput (PLD policy, cap_i = the
// proposal lengths just written) -- GetVerificationLen right after Propose (Listing 1).
//
// READY (TSV_LOOKUP_INPUTS_READY, include/tsv.h): no kernel still in flight writes the inputs or reads
// the outputs, so the whole kernel -- the search, the stores of the proposals and, when FUSED, the
// batch sums, the last CTA's ArgMaxGoodput and its stores -- runs before the grid-dependency wait,
// overlapping the preceding kernel; every thread waits at the very end, so the kernel still completes
// after its predecessor and triggers its dependents only after its own wait (the PDL chain invariant).
template <bool FUSED, bool READY = false>
__global__ void __launch_bounds__(kLookupThreads)
    ngram_lookup_kernel(const int32_t* __restrict__ ctx, const int32_t* __restrict__ ctx_offsets, int32_t B,
                        int32_t n_min, int32_t n_max, int32_t K, int32_t* __restrict__ proposals,
                        int32_t* __restrict__ proposal_len, ChooseArgs ca, uint32_t* counter, int32_t* devstatus) {
    __shared__ uint32_t s_red[kLookupThreads / 32];
    TSV_STEP_SPAN(0);
    if (!READY) {
        pdl_wait();
        TSV_STEP_WAITED();
        pdl_launch_dependents();
    }
    const int32_t i = blockIdx.x;
    const int tid = threadIdx.x;
    const int32_t off = __ldg(ctx_offsets + i);
    const int32_t end = __ldg(ctx_offsets + i + 1);
    // device-side data errors (tsv.h): offsets negative or decreasing, or L_i > TSV_MAX_CONTEXT (the
    // packed key holds e in 20 bits) -> no proposal and TSV_DEVSTATUS_BAD_CONTEXT
    const int64_t L64 = static_cast<int64_t>(end) - off;
    const bool bad_ctx = off < 0 || L64 < 0 || L64 > TSV_MAX_CONTEXT;
    const int32_t L = bad_ctx ? 0 : static_cast<int32_t>(L64);
    if (!READY && bad_ctx && tid == 0 && devstatus) atomicOr(reinterpret_cast<unsigned int*>(devstatus), TSV_DEVSTATUS_BAD_CONTEXT);
    const int32_t* c = ctx + off;
    int32_t my_len = 0;  // this request's proposal length (warp 0)
    uint32_t best = 0;
    if (L >= 2) {
        const int64_t last = static_cast<int64_t>(off) + L - 1;
        Query Q;
        Q.q0 = __ldg(ctx + last);
        Q.q1 = __ldg(ctx + last - 1);
        Q.q2 = L >= 3 ? __ldg(ctx + last - 2) : 0;
        Q.q3 = L >= 4 ? __ldg(ctx + last - 3) : 0;
        Q.off = off;
        Q.L = L;
        Q.n_max = n_max;
        const bool vec = (reinterpret_cast<uintptr_t>(ctx) & 15u) == 0;
        const int64_t g_lo = off >> 2, g_hi = (last - 1) >> 2;  // groups holding e in [0, L-2]
        for (int64_t g0 = g_lo + tid; g0 <= g_hi; g0 += kLookupUnroll * kLookupThreads) {
            Group G[kLookupUnroll];
#pragma unroll
            for (int u = 0; u < kLookupUnroll; ++u) {
                const int64_t g = g0 + u * kLookupThreads;
                if (g <= g_hi) G[u] = load_group(ctx, g, last, vec);
            }
#pragma unroll
            for (int u = 0; u < kLookupUnroll; ++u) {
                const int64_t g = g0 + u * kLookupThreads;
                if (g <= g_hi) {
                    const uint32_t k = scan_group(ctx, G[u], g, Q);
                    best = k > best ? k : best;
                }
            }
        }
    }
    best = __reduce_max_sync(0xFFFFFFFFu, best);
    if ((tid & 31) == 0) s_red[tid >> 5] = best;
    __syncthreads();
    if (tid < 32) {
        uint32_t v = tid < kLookupThreads / 32 ? s_red[tid] : 0u;
        v = __reduce_max_sync(0xFFFFFFFFu, v);
        const int32_t n_star = static_cast<int32_t>(v >> 20);
        const int32_t e_star = static_cast<int32_t>(v & 0xFFFFFu);
        int32_t len = 0;
        if (L >= 2 && n_star >= n_min) len = min(K, L - 1 - e_star);
        my_len = len;
        int32_t* out = proposals + static_cast<int64_t>(i) * K;
        for (int32_t t = tid; t < K; t += 32) out[t] = t < len ? __ldg(c + e_star + 1 + t) : -1;
        if (tid == 0) {
            proposal_len[i] = len;
            if (READY && bad_ctx && devstatus) atomicOr(reinterpret_cast<unsigned int*>(devstatus), TSV_DEVSTATUS_BAD_CONTEXT);
        }
    }
    if (FUSED) fused_choose_k(ca, reinterpret_cast<FusedScratch*>(counter), i, my_len);
    if (READY) {
        pdl_wait();
        TSV_STEP_WAITED();
        pdl_launch_dependents();
    }
}

}  // namespace tsv

using namespace tsv;
TSV_STEP_TRACE_READER(lookup)

extern "C" tsv_status tsv_propose_lookup(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                                         int32_t n_min, int32_t n_max, int32_t k_fixed,
                                         int32_t* proposals, int32_t* proposal_len, int32_t* device_status,
                                         void* stream) {
    TSV_TRACE_CALL();
    return tsv_propose_lookup_ex(ctx, ctx_offsets, B, n_min, n_max, k_fixed, proposals, proposal_len, device_status,
                                 0, stream);
}

extern "C" tsv_status tsv_propose_lookup_ex(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                                            int32_t n_min, int32_t n_max, int32_t k_fixed,
                                            int32_t* proposals, int32_t* proposal_len, int32_t* device_status,
                                            int32_t flags, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE((flags & ~TSV_LOOKUP_INPUTS_READY) == 0, "tsv_propose_lookup: unknown flags 0x%x", flags);
    TSV_REQUIRE(B >= 0, "tsv_propose_lookup: B < 0 (%d)", B);
    TSV_REQUIRE(n_min >= 1 && n_min <= n_max && n_max <= TSV_MAX_NGRAM,
                "tsv_propose_lookup: need 1 <= n_min (%d) <= n_max (%d) <= %d", n_min, n_max, TSV_MAX_NGRAM);
    TSV_REQUIRE(k_fixed >= 1 && k_fixed <= TSV_MAX_K, "tsv_propose_lookup: k_fixed %d outside [1, %d]", k_fixed, TSV_MAX_K);
    if (B == 0) return TSV_OK;
    TSV_REQUIRE(ctx && ctx_offsets && proposals && proposal_len, "tsv_propose_lookup: a required array is NULL");
    TSV_TRY(check_device());
    ChooseArgs none = {};
    auto kern = (flags & TSV_LOOKUP_INPUTS_READY) ? ngram_lookup_kernel<false, true> : ngram_lookup_kernel<false, false>;
    TSV_CUDA(launch_pdl(kern, dim3(B), dim3(kLookupThreads), 0,
                        static_cast<cudaStream_t>(stream), ctx, ctx_offsets, B, n_min, n_max, k_fixed, proposals,
                        proposal_len, none, static_cast<uint32_t*>(nullptr), device_status),
             "ngram_lookup_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_propose_lookup_choose_k(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                                                  int32_t n_min, int32_t n_max, int32_t k_fixed,
                                                  int32_t* proposals, int32_t* proposal_len,
                                                  const double* alpha, int32_t alpha_per_request,
                                                  const int32_t* ctx_len, tsv_latency_model target,
                                                  double pld_cost_ms, int64_t kv_free_slots, int32_t* k_out,
                                                  double* goodput_out, int32_t* k_per_request,
                                                  uint32_t* counter, int32_t* device_status, void* stream) {
    TSV_TRACE_CALL();
    return tsv_propose_lookup_choose_k_ex(ctx, ctx_offsets, B, n_min, n_max, k_fixed, proposals, proposal_len, alpha,
                                          alpha_per_request, ctx_len, target, pld_cost_ms, kv_free_slots, k_out,
                                          goodput_out, k_per_request, counter, device_status, nullptr, 0, stream);
}

extern "C" tsv_status tsv_propose_lookup_choose_k_ex(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                                                     int32_t n_min, int32_t n_max, int32_t k_fixed,
                                                     int32_t* proposals, int32_t* proposal_len,
                                                     const double* alpha, int32_t alpha_per_request,
                                                     const int32_t* ctx_len, tsv_latency_model target,
                                                     double pld_cost_ms, int64_t kv_free_slots, int32_t* k_out,
                                                     double* goodput_out, int32_t* k_per_request,
                                                     uint32_t* counter, int32_t* device_status,
                                                     const uint32_t* alpha_ready, int32_t flags, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE((flags & ~TSV_LOOKUP_INPUTS_READY) == 0, "tsv_propose_lookup_choose_k: unknown flags 0x%x", flags);
    TSV_REQUIRE(B >= 1, "tsv_propose_lookup_choose_k: B must be >= 1 (got %d)", B);
    TSV_REQUIRE(n_min >= 1 && n_min <= n_max && n_max <= TSV_MAX_NGRAM,
                "tsv_propose_lookup_choose_k: need 1 <= n_min (%d) <= n_max (%d) <= %d", n_min, n_max, TSV_MAX_NGRAM);
    TSV_REQUIRE(k_fixed >= 1 && k_fixed <= TSV_MAX_K, "tsv_propose_lookup_choose_k: k_fixed %d outside [1, %d]", k_fixed, TSV_MAX_K);
    TSV_REQUIRE(ctx && ctx_offsets && proposals && proposal_len && alpha && ctx_len && k_out,
                "tsv_propose_lookup_choose_k: a required array is NULL");
    TSV_REQUIRE_WS(counter != nullptr, "tsv_propose_lookup_choose_k: scratch (counter) is NULL");
    TSV_REQUIRE((reinterpret_cast<uintptr_t>(counter) & 7u) == 0, "tsv_propose_lookup_choose_k: scratch must be 8-byte aligned");
    TSV_TRY(check_device());
    ChooseArgs A = {};
    A.alpha = alpha;
    A.ctx_len = ctx_len;
    A.cap = proposal_len;
    A.k_out = k_out;
    A.goodput_out = goodput_out;
    A.k_per_request = k_per_request;
    A.target = target;
    A.draft = target;
    A.pld_cost_ms = pld_cost_ms;
    A.kv_free = static_cast<long long>(kv_free_slots);
    A.alpha_ready = alpha_ready;
    A.devstatus = device_status;
    A.alpha_per_request = alpha_per_request;
    A.B = B;
    A.k_max = k_fixed;
    A.policy = TSV_POLICY_PLD;
    auto kern = (flags & TSV_LOOKUP_INPUTS_READY) ? ngram_lookup_kernel<true, true> : ngram_lookup_kernel<true, false>;
    TSV_CUDA(launch_pdl(kern, dim3(B), dim3(kLookupThreads), 0,
                        static_cast<cudaStream_t>(stream), ctx, ctx_offsets, B, n_min, n_max, k_fixed, proposals,
                        proposal_len, A, counter, device_status),
             "ngram_lookup_kernel launch");
    return TSV_OK;
}
