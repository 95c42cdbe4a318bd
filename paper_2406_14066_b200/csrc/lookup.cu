// lookup.cu -- prompt-lookup n-gram proposal (PLD) on sm_100a (K2).
// PAPER.md:57 [AD] (fixed-length proposal; cost depends only on the context search),
// PAPER.md:454, 498 (n-grams retrieved from the prompt), Fig. PAPER.md:44-49
// (a request with no match proposes nothing); reading R20 in DESIGN.md section 3.
//
// "Longest n in [n_min, n_max] with a match, then the latest start" is evaluated as
// ONE max-reduction: for every end position e in [0, L-2] let c(e)
// be the length of the common suffix of ctx[..e] and ctx[..L-1] capped at n_max;
// key(e) = (c(e) << 20) | e.  The lexicographic max of (c, e) is exactly the longest
// matching n and, among its matches, the latest one.  One CTA per request: the context
// is staged into shared memory with a TMA bulk copy (cp.async.bulk) when it fits,
// each thread scores a strided set of end positions against the query suffix held in
// registers, and a warp REDUX + shared-memory step reduces the keys.
#include "goodput.cuh"

namespace tsv {

constexpr int kLookupThreads = 256;
constexpr int kLookupSmemInts = 11008;  // 43 KB static smem: contexts up to ~11K tokens are staged

// FUSED: the CTA that finishes last also runs ArgMaxGoodput (PLD policy, cap_i = the
// proposal lengths just written) -- GetVerificationLen right after Propose (Listing 1).
template <bool FUSED>
__global__ void __launch_bounds__(kLookupThreads)
    ngram_lookup_kernel(const int32_t* __restrict__ ctx, const int32_t* __restrict__ ctx_offsets, int32_t B,
                        int32_t n_min, int32_t n_max, int32_t K, int32_t* __restrict__ proposals,
                        int32_t* __restrict__ proposal_len, ChooseArgs ca, uint32_t* counter) {
    __shared__ __align__(128) int32_t s_ctx[kLookupSmemInts];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint32_t s_red[kLookupThreads / 32];
    pdl_wait();
    pdl_launch_dependents();
    const int32_t i = blockIdx.x;
    const int32_t off = ctx_offsets[i];
    const int32_t L = ctx_offsets[i + 1] - off;
    const int32_t* c = ctx + off;
    const int tid = threadIdx.x;

    // ---- stage the context: aligned middle by one TMA bulk copy, ragged edges by LDG
    const bool staged = L > 0 && L <= kLookupSmemInts - 8 && (reinterpret_cast<uintptr_t>(ctx) & 15u) == 0;
    int32_t shift = 0;  // s_ctx[shift + t] == c[t]; shift = off & 3 keeps int4 groups aligned
    if (staged) {
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(c);
        const uintptr_t a_lo = (a0 + 15) & ~static_cast<uintptr_t>(15);         // first aligned byte inside
        const uintptr_t a_hi = (a0 + 4ull * L) & ~static_cast<uintptr_t>(15);   // last aligned byte inside
        const int32_t head = static_cast<int32_t>((a_lo - a0) >> 2);            // elements before a_lo
        shift = (4 - head) & 3;  // so that s_ctx + shift + head is 16-byte aligned
        const bool has_mid = a_hi > a_lo;
        const uint32_t mid_bytes = has_mid ? static_cast<uint32_t>(a_hi - a_lo) : 0u;
        if (tid == 0) {
            mbar_init(&s_bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0 && has_mid) {
            mbar_expect_tx(&s_bar, mid_bytes);
            bulk_g2s(s_ctx + shift + head, reinterpret_cast<const void*>(a_lo), mid_bytes, &s_bar);
        }
        const int32_t mid_elems = static_cast<int32_t>(mid_bytes >> 2);
        const int32_t n_head = min(head, L);              // ragged edges by plain loads
        const int32_t tail0 = head + mid_elems;
        if (tid < n_head) s_ctx[shift + tid] = c[tid];
        if (has_mid && tail0 + tid < L) s_ctx[shift + tail0 + tid] = c[tail0 + tid];
        if (!has_mid)
            for (int32_t t = n_head + tid; t < L; t += kLookupThreads) s_ctx[shift + t] = c[t];
        if (has_mid) mbar_wait(&s_bar, 0);
        __syncthreads();
    }
    const int32_t* src = staged ? (s_ctx + shift) : c;

    // ---- key(e) = (min(c(e), n_max) << 20) | e over e in [0, L-2]; c(e) = common suffix
    // length of ctx[..e] and ctx[..L-1].  Fast path: compare ctx[e] with the last token q0
    // four positions at a time; only on a hit is the rest of the suffix compared.
    uint32_t best = 0;
    if (L >= 2) {
        const int32_t q0 = src[L - 1];
        auto suffix_key = [&](int32_t e) -> uint32_t {  // ctx[e] == q0 already
            int32_t cl = 1;
            while (cl < n_max && cl <= e && src[e - cl] == src[L - 1 - cl]) ++cl;
            return (static_cast<uint32_t>(cl) << 20) | static_cast<uint32_t>(e);
        };
        if (staged) {
            const int4* s4 = reinterpret_cast<const int4*>(s_ctx);
            const int32_t n_groups = (shift + L - 1 + 3) >> 2;  // smem ints [0, shift + L - 1) hold e <= L-2
            for (int32_t g = tid; g < n_groups; g += kLookupThreads) {
                const int4 v = s4[g];
                const int32_t e0 = 4 * g - shift;
                const int32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const int32_t e = e0 + s;
                    if (vv[s] == q0 && e >= 0 && e <= L - 2) {
                        const uint32_t key = suffix_key(e);
                        best = key > best ? key : best;
                    }
                }
            }
        } else {
            for (int32_t e = tid; e <= L - 2; e += kLookupThreads) {
                if (src[e] == q0) {
                    const uint32_t key = suffix_key(e);
                    best = key > best ? key : best;
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
        int32_t* out = proposals + static_cast<int64_t>(i) * K;
        for (int32_t t = tid; t < K; t += 32) out[t] = t < len ? src[e_star + 1 + t] : -1;
        if (tid == 0) proposal_len[i] = len;
    }
    if (FUSED && last_cta_done(counter, static_cast<uint32_t>(B))) choose_k_block(ca);
}

}  // namespace tsv

using namespace tsv;

extern "C" tsv_status tsv_propose_lookup(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                                         int32_t n_min, int32_t n_max, int32_t k_fixed,
                                         int32_t* proposals, int32_t* proposal_len, void* stream) {
    TSV_REQUIRE(B >= 0, "tsv_propose_lookup: B < 0 (%d)", B);
    TSV_REQUIRE(n_min >= 1 && n_min <= n_max && n_max <= TSV_MAX_NGRAM,
                "tsv_propose_lookup: need 1 <= n_min (%d) <= n_max (%d) <= %d", n_min, n_max, TSV_MAX_NGRAM);
    TSV_REQUIRE(k_fixed >= 1 && k_fixed <= TSV_MAX_K, "tsv_propose_lookup: k_fixed %d outside [1, %d]", k_fixed, TSV_MAX_K);
    if (B == 0) return TSV_OK;
    TSV_REQUIRE(ctx && ctx_offsets && proposals && proposal_len, "tsv_propose_lookup: a required array is NULL");
    TSV_TRY(check_device());
    ChooseArgs none = {};
    TSV_CUDA(launch_pdl(ngram_lookup_kernel<false>, dim3(B), dim3(kLookupThreads), 0, static_cast<cudaStream_t>(stream),
                        ctx, ctx_offsets, B, n_min, n_max, k_fixed, proposals, proposal_len, none,
                        static_cast<uint32_t*>(nullptr)),
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
                                                  uint32_t* counter, void* stream) {
    TSV_REQUIRE(B >= 1, "tsv_propose_lookup_choose_k: B must be >= 1 (got %d)", B);
    TSV_REQUIRE(n_min >= 1 && n_min <= n_max && n_max <= TSV_MAX_NGRAM,
                "tsv_propose_lookup_choose_k: need 1 <= n_min (%d) <= n_max (%d) <= %d", n_min, n_max, TSV_MAX_NGRAM);
    TSV_REQUIRE(k_fixed >= 1 && k_fixed <= TSV_MAX_K, "tsv_propose_lookup_choose_k: k_fixed %d outside [1, %d]", k_fixed, TSV_MAX_K);
    TSV_REQUIRE(ctx && ctx_offsets && proposals && proposal_len && alpha && ctx_len && k_out && counter,
                "tsv_propose_lookup_choose_k: a required array is NULL");
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
    A.alpha_per_request = alpha_per_request;
    A.B = B;
    A.k_max = k_fixed;
    A.policy = TSV_POLICY_PLD;
    TSV_CUDA(launch_pdl(ngram_lookup_kernel<true>, dim3(B), dim3(kLookupThreads), 0, static_cast<cudaStream_t>(stream),
                        ctx, ctx_offsets, B, n_min, n_max, k_fixed, proposals, proposal_len, A, counter),
             "ngram_lookup_kernel launch");
    return TSV_OK;
}
