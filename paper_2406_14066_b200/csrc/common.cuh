// common.cuh -- internals shared by the sm_100a kernels of libtsv (not part of the ABI).
//
// Philox4x32-10 (Salmon et al., SC'11), the race / acceptance uniforms and the
// packed argmax key, as fixed by DESIGN.md readings R2, R6-R9.  Independent of
// oracle/ (which has its own implementation of the same published definitions).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tsv.h"
#include <nvtx3/nvToolsExt.h>

namespace tsv {

// ---------------------------------------------------------------- host side
void set_error(const char* fmt, ...);
tsv_status check_device();                       // sm_100 only
tsv_status cuda_status(cudaError_t e, const char* what);

#define TSV_REQUIRE(cond, ...)                         \
    do {                                               \
        if (!(cond)) {                                 \
            ::tsv::set_error(__VA_ARGS__);             \
            return TSV_ERR_INVALID_ARG;                \
        }                                              \
    } while (0)

// workspace NULL or smaller than required (TSV_ERR_WORKSPACE, tsv.h)
#define TSV_REQUIRE_WS(cond, ...)                      \
    do {                                               \
        if (!(cond)) {                                 \
            ::tsv::set_error(__VA_ARGS__);             \
            return TSV_ERR_WORKSPACE;                  \
        }                                              \
    } while (0)

#define TSV_CUDA(call, what)                                               \
    do {                                                                   \
        cudaError_t e__ = (call);                                          \
        if (e__ != cudaSuccess) return ::tsv::cuda_status(e__, what);      \
    } while (0)

#define TSV_TRY(call)                                  \
    do {                                               \
        tsv_status s__ = (call);                       \
        if (s__ != TSV_OK) return s__;                 \
    } while (0)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Tracing: with TSV_NVTX=1 in the environment every C-ABI entry point opens an
// NVTX range named after itself (host side: the call that enqueues the kernels), visible to nsys and to
// ncu's --nvtx filters.  Off by default; one cached getenv per process.
bool nvtx_enabled();
struct NvtxScope {
    bool on;
    explicit NvtxScope(const char* name) : on(nvtx_enabled()) {
        if (on) nvtxRangePushA(name);
    }
    ~NvtxScope() {
        if (on) nvtxRangePop();
    }
};
#define TSV_TRACE_CALL() ::tsv::NvtxScope tsv_nvtx_scope_(__func__)

// ---------------------------------------------------------------- device side
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

constexpr uint32_t kPurposeAccept = 0u;
constexpr uint32_t kPurposeRace = 1u;

// Philox4x32-10.  The key schedule depends only on the seed (kernel-uniform),
// and for the race c1..c3 are row-uniform, so ptxas hoists the first round's
// second product and the second round's first product out of vocab loops.
__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(kPhiloxM0, c0);
        const uint32_t lo0 = kPhiloxM0 * c0;
        const uint32_t hi1 = __umulhi(kPhiloxM1, c2);
        const uint32_t lo1 = kPhiloxM1 * c2;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    return make_uint4(c0, c1, c2, c3);
}

// u_acc = (x >> 8) 2^-24 in [0, 1): exact in binary32.
__device__ __forceinline__ float u_acc_from_word(uint32_t x) {
    return __uint2float_rn(x >> 8) * 0x1p-24f;
}

// The race uniform is u_race = (2 (x & 0x7FFFFF) + 1) 2^-24 in (0, 1), exact in binary32 (R7);
// the kernels only ever need 1 - u_race, exactly, with one LOP3 and one FADD:
// as_float((x & 0x7FFFFF) ^ 0x3FFFFFFF) = 2 - (m+1) 2^-23 with m = x & 0x7FFFFF, and
// subtracting (1 - 2^-24) leaves 1 - (2m+1) 2^-24 (24 significant bits: exact).
__device__ __forceinline__ float one_minus_u_race(uint32_t x) {
    uint32_t b;  // (x & 0x7FFFFF) ^ 0x3FFFFFFF as ONE lop3 (ptxas otherwise emits two)
    asm("lop3.b32 %0, %1, 0x7FFFFF, %2, 0x6A;" : "=r"(b) : "r"(x), "r"(0x3FFFFFFFu));
    return __fsub_rn(__uint_as_float(b), 0x1.fffffep-1f);
}

// 32x32 -> 64-bit product as one IMAD.WIDE.U32: returns lo, writes hi.
__device__ __forceinline__ uint32_t mulhilo(uint32_t a, uint32_t m, uint32_t& hi) {
    const unsigned long long p = static_cast<unsigned long long>(a) * m;
    hi = static_cast<uint32_t>(p >> 32);
    return static_cast<uint32_t>(p);
}

// Philox4x32-10 for the race of one row: counter (quad, c1, c2, c3) with c1..c3 fixed
// for the row.  Rounds 1-3 fold the row-uniform products and xors into constants
// computed once per row (RaceCtr), leaving 2 + 3 + 4 + 7*4 = 37 ops per quad.
struct RaceCtr {
    uint32_t u0, u1;   // round-1 outputs c0', c1' (depend only on c1, c2, k0)
    uint32_t k1a;      // c3 ^ k1
    uint32_t k0b;      // u1 ^ (k0 + W0)
    uint32_t k1b;      // hi(M0 u0) ^ (k1 + W1)
    uint32_t l0;       // lo(M0 u0)
    uint32_t k1c;      // l0 ^ (k1 + 2 W1)
};

__device__ __forceinline__ RaceCtr race_ctr(uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
    RaceCtr r;
    const uint32_t hi1 = __umulhi(kPhiloxM1, c2), lo1 = kPhiloxM1 * c2;
    r.u0 = hi1 ^ c1 ^ k0;
    r.u1 = lo1;
    r.k1a = c3 ^ k1;
    const uint32_t H0 = __umulhi(kPhiloxM0, r.u0), L0 = kPhiloxM0 * r.u0;
    r.k0b = r.u1 ^ (k0 + kPhiloxW0);
    r.k1b = H0 ^ (k1 + kPhiloxW1);
    r.l0 = L0;
    r.k1c = L0 ^ (k1 + 2u * kPhiloxW1);
    return r;
}

// ks0[r] = k0 + r W0, ks1[r] = k1 + r W1: the key schedule, precomputed on the host and
// passed in the kernel parameter block so every xor reads it from the constant bank.
template <typename KS>
__device__ __forceinline__ uint4 philox_race(const RaceCtr& r, uint32_t quad, const KS& ks) {
    uint32_t hi0, hi1;
    // round 1
    uint32_t c3 = mulhilo(quad, kPhiloxM0, hi0);
    uint32_t c2 = hi0 ^ r.k1a;
    // round 2 (c0 = u0 is row-uniform: its product is r.k1b / r.l0)
    uint32_t lo1 = mulhilo(c2, kPhiloxM1, hi1);
    uint32_t c0 = hi1 ^ r.k0b;
    uint32_t c1 = lo1;
    c2 = r.k1b ^ c3;
    // round 3 (its c3 input is r.l0)
    {
        const uint32_t lo0 = mulhilo(c0, kPhiloxM0, hi0);
        lo1 = mulhilo(c2, kPhiloxM1, hi1);
        c0 = hi1 ^ c1 ^ ks.ks0[2];
        c1 = lo1;
        c2 = hi0 ^ r.k1c;
        c3 = lo0;
    }
#pragma unroll
    for (int rr = 3; rr < 10; ++rr) {
        const uint32_t lo0 = mulhilo(c0, kPhiloxM0, hi0);
        lo1 = mulhilo(c2, kPhiloxM1, hi1);
        const uint32_t n0 = hi1 ^ c1 ^ ks.ks0[rr];
        const uint32_t n2 = hi0 ^ c3 ^ ks.ks1[rr];
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

// E(u) = RN32(-ln u) (R9).  Any double evaluation within a few ulp of -ln u rounds to the
// same binary32 value: every race uniform keeps >= 74 double-ulp from a binary32 midpoint
// (oracle pin; GPU-checked exhaustively).  Near u = 1 -- where the race's survivors live --
// -ln u = -log1p(-x), x = 1 - u exact, is summed as x + x^2/2 + ... + x^8/8 by Horner
// (truncation < x^8/9 relative <= 2^-51 for x < 2^-6); elsewhere the CUDA double log.
__device__ __forceinline__ float race_E_omu(float omu) {
    const double x = static_cast<double>(omu);
    if (omu < 0x1p-6f) {
        double s = 1.0 / 8.0;
        s = __fma_rn(s, x, 1.0 / 7.0);
        s = __fma_rn(s, x, 1.0 / 6.0);
        s = __fma_rn(s, x, 1.0 / 5.0);
        s = __fma_rn(s, x, 1.0 / 4.0);
        s = __fma_rn(s, x, 1.0 / 3.0);
        s = __fma_rn(s, x, 0.5);
        s = __fma_rn(s, x, 1.0);
        return __double2float_rn(__dmul_rn(s, x));
    }
    return __double2float_rn(-log(1.0 - x));
}
__device__ __forceinline__ float race_E(float u) {
    return __double2float_rn(-log(static_cast<double>(u)));
}

// Packed argmax key: score bits (non-negative binary32 orders like uint32)
// above the complemented global index, so max(key) = max score, lowest index.
__device__ __forceinline__ uint64_t pack_key(float s, uint32_t v_global) {
    return (static_cast<uint64_t>(__float_as_uint(s)) << 32) | static_cast<uint64_t>(0xFFFFFFFFu - v_global);
}
__device__ __forceinline__ int32_t key_index(uint64_t key) {
    return static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(key & 0xFFFFFFFFu));
}

// Exact race key of one element with weight w > 0 and Philox word x.
__device__ __forceinline__ uint64_t exact_race_key(float w, uint32_t x, uint32_t v_global) {
    const float E = race_E_omu(one_minus_u_race(x));
    return pack_key(__fdiv_rn(w, E), v_global);
}

// F = 1 - u + (1 - 2^-24) in [1, 2): the float bits (x & 0x7FFFFF) ^ 0x3FFFFFFF, one LOP3.
__device__ __forceinline__ float race_F(uint32_t x) {
    uint32_t b;
    asm("lop3.b32 %0, %1, 0x7FFFFF, %2, 0x6A;" : "=r"(b) : "r"(x), "r"(0x3FFFFFFFu));
    return __uint_as_float(b);
}

// Warp-wide max of a u64 (all lanes): the max high word by one REDUX, then the max low word among the
// lanes holding it by a second -- the same value as the lexicographic max, in two reductions instead of
// five rounds of 64-bit shuffles.
#ifndef TSV_WARP_MAX_REDUX
#define TSV_WARP_MAX_REDUX 1
#endif
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
    if (!TSV_WARP_MAX_REDUX) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t t = __shfl_xor_sync(0xFFFFFFFFu, v, o);
            v = t > v ? t : v;
        }
        return v;
    }
    const uint32_t hi = static_cast<uint32_t>(v >> 32), lo = static_cast<uint32_t>(v);
    const uint32_t mhi = __reduce_max_sync(0xFFFFFFFFu, hi);
    const uint32_t mlo = __reduce_max_sync(0xFFFFFFFFu, hi == mhi ? lo : 0u);
    return (static_cast<uint64_t>(mhi) << 32) | mlo;
}

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of a step is launched with programmaticStreamSerialization: it may start
// while its predecessor drains, runs its prologue, and blocks in griddepcontrol.wait
// before touching data the predecessor produced (full completion + visibility).
// OR status bits into the caller's device_status word (nullable).
__device__ __forceinline__ void report(int32_t* devstatus, uint32_t bits) {
    if (devstatus && bits) atomicOr(reinterpret_cast<unsigned int*>(devstatus), bits);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Step timeline (diagnostic builds only, -DTSV_STEP_TRACE=1; scripts/diag_step_trace.py): thread 0 of
// every CTA of the step's kernels records (kernel id, CTA, entry, after the grid-dependency wait, exit)
// from %globaltimer into its translation unit's buffer (read by tsv_debug_step_trace_*).
#ifndef TSV_STEP_TRACE
#define TSV_STEP_TRACE 0
#endif
#if TSV_STEP_TRACE
constexpr unsigned kStepTraceMax = 1u << 16;
static __device__ unsigned long long g_step_tr[kStepTraceMax][6];
static __device__ unsigned int g_step_tr_n;
__device__ __forceinline__ unsigned long long step_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
struct StepTrace {
    unsigned long long t0, t1, m1, m2;
    int id;
    __device__ explicit StepTrace(int i) : t0(step_ns()), t1(0), m1(0), m2(0), id(i) {}
    __device__ void waited() { t1 = step_ns(); }
    __device__ void mark(int n) { (n == 1 ? m1 : m2) = step_ns(); }
    __device__ ~StepTrace() {
        if (threadIdx.x == 0) {
            const unsigned k = atomicAdd(&g_step_tr_n, 1u);
            if (k < kStepTraceMax) {
                g_step_tr[k][0] = (static_cast<unsigned long long>(blockIdx.x) << 8) | static_cast<unsigned>(id);
                g_step_tr[k][1] = t0;
                g_step_tr[k][2] = t1;
                g_step_tr[k][3] = step_ns();
                g_step_tr[k][4] = m1;
                g_step_tr[k][5] = m2;
            }
        }
    }
};
#define TSV_STEP_SPAN(id) ::tsv::StepTrace tsv_step_span_(id)
#define TSV_STEP_WAITED() tsv_step_span_.waited()
#define TSV_STEP_MARK(n) tsv_step_span_.mark(n)
#define TSV_STEP_TRACE_READER(name)                                                                   \
    extern "C" TSV_API unsigned tsv_debug_step_trace_##name(unsigned long long* out, unsigned max_n) { \
        unsigned n = 0;                                                                               \
        cudaMemcpyFromSymbol(&n, ::tsv::g_step_tr_n, sizeof(n));                                      \
        n = n < max_n ? n : max_n;                                                                    \
        if (n > ::tsv::kStepTraceMax) n = ::tsv::kStepTraceMax;                                       \
        cudaMemcpyFromSymbol(out, ::tsv::g_step_tr, n * 6 * sizeof(unsigned long long));              \
        unsigned z = 0;                                                                               \
        cudaMemcpyToSymbol(::tsv::g_step_tr_n, &z, sizeof(z));                                        \
        return n;                                                                                     \
    }
#else
#define TSV_STEP_SPAN(id) \
    do {                  \
    } while (0)
#define TSV_STEP_WAITED() \
    do {                  \
    } while (0)
#define TSV_STEP_MARK(n) \
    do {                 \
    } while (0)
#define TSV_STEP_TRACE_READER(name)
#endif
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

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
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace tsv
