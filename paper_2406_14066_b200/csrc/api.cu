// api.cu -- error reporting, device gating and the NCCL communicator of libtsv.
//
// NCCL is resolved at run time (dlopen of the process's libnccl.so.2, normally the
// copy torch already loaded) so the library has no link-time NCCL dependency and a
// single-GPU process never touches it.  The multi-GPU modes:
//   request-sharded: no data-path collective; tsv_allreduce_i64 sums the int64
//                    fixed-point goodput / acceptance counters across ranks;
//   vocab-sharded:   tsv_verify_accept_sharded = shard partial -> ncclAllGather of
//                    tsv_shard_tuple rows over NVLink/NVSwitch -> combine.
#include <stdlib.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "common.cuh"

namespace tsv {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

tsv_status cuda_status(cudaError_t e, const char* what) {
    set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    return TSV_ERR_CUDA;
}

bool nvtx_enabled() {
    static const bool on = [] {
        const char* e = getenv("TSV_NVTX");
        return e && e[0] == '1';
    }();
    return on;
}

tsv_status check_device() {
    static int cached[64];  // 0 unknown, 1 ok, 2 unsupported
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    if (dev >= 0 && dev < 64 && cached[dev] == 1) return TSV_OK;
    int major = 0, minor = 0;
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
    e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
    const bool ok = major == 10 && minor == 0;
    if (dev >= 0 && dev < 64) cached[dev] = ok ? 1 : 2;
    if (!ok) {
        set_error("device %d is sm_%d%d; libtsv is built for sm_100a (B200) only", dev, major, minor);
        return TSV_ERR_UNSUPPORTED_DEVICE;
    }
    return TSV_OK;
}

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    const char* (*GetErrorString)(ncclResult_t);
    bool ok;
};

static NcclApi g_nccl;
static std::once_flag g_nccl_once;

static void load_nccl() {
    memset(&g_nccl, 0, sizeof(g_nccl));
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define TSV_SYM(field, name) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name))
    TSV_SYM(GetUniqueId, "ncclGetUniqueId");
    TSV_SYM(CommInitRank, "ncclCommInitRank");
    TSV_SYM(CommDestroy, "ncclCommDestroy");
    TSV_SYM(AllGather, "ncclAllGather");
    TSV_SYM(AllReduce, "ncclAllReduce");
    TSV_SYM(GetErrorString, "ncclGetErrorString");
#undef TSV_SYM
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllGather &&
                g_nccl.AllReduce && g_nccl.GetErrorString;
}

static tsv_status nccl_ready() {
    std::call_once(g_nccl_once, load_nccl);
    if (!g_nccl.ok) {
        set_error("NCCL (libnccl.so.2) could not be loaded");
        return TSV_ERR_NCCL;
    }
    return TSV_OK;
}

static tsv_status nccl_status(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return TSV_OK;
    set_error("%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error");
    return TSV_ERR_NCCL;
}

}  // namespace tsv

struct tsv_comm {
    ncclComm_t comm;
    int32_t rank, world;
};

using namespace tsv;

extern "C" const char* tsv_last_error(void) { return g_err; }
extern "C" int tsv_abi_version(void) { return TSV_ABI_VERSION; }

extern "C" tsv_status tsv_comm_get_unique_id(void* unique_id_out) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(unique_id_out != nullptr, "tsv_comm_get_unique_id: out is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    TSV_TRY(nccl_ready());
    ncclUniqueId id;
    TSV_TRY(nccl_status(g_nccl.GetUniqueId(&id), "ncclGetUniqueId"));
    memcpy(unique_id_out, &id, sizeof(id));
    return TSV_OK;
}

extern "C" tsv_status tsv_comm_init(tsv_comm** out, const void* unique_id, int32_t rank, int32_t world) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(out && unique_id, "tsv_comm_init: NULL argument");
    TSV_REQUIRE(world >= 1 && rank >= 0 && rank < world, "tsv_comm_init: bad rank %d / world %d", rank, world);
    TSV_TRY(check_device());
    TSV_TRY(nccl_ready());
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    tsv_comm* c = new tsv_comm();
    c->rank = rank;
    c->world = world;
    tsv_status s = nccl_status(g_nccl.CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
    if (s != TSV_OK) {
        delete c;
        return s;
    }
    *out = c;
    return TSV_OK;
}

extern "C" tsv_status tsv_comm_destroy(tsv_comm* comm) {
    TSV_TRACE_CALL();
    if (!comm) return TSV_OK;
    TSV_TRY(nccl_ready());
    tsv_status s = nccl_status(g_nccl.CommDestroy(comm->comm), "ncclCommDestroy");
    delete comm;
    return s;
}

// Sharded workspace: [verify slots][dense: tuples local + gathered G x rows_p | lazy: masks B, keys 2B]
extern "C" tsv_status tsv_verify_sharded_workspace_size(const tsv_verify_args* a, int32_t world, size_t* bytes) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(a && bytes, "tsv_verify_sharded_workspace_size: NULL argument");
    TSV_REQUIRE(world >= 1, "tsv_verify_sharded_workspace_size: world < 1");
    size_t slots = 0;
    TSV_TRY(tsv_verify_workspace_size(a, &slots));
    const size_t rows = static_cast<size_t>(a->rows_p);
    slots = (slots + 255) & ~static_cast<size_t>(255);
    const size_t dense = rows * sizeof(tsv_shard_tuple) * (1 + static_cast<size_t>(world));
    const size_t lazy = 3 * sizeof(uint64_t) * static_cast<size_t>(a->B);
    *bytes = slots + (dense > lazy ? dense : lazy);
    return TSV_OK;
}

extern "C" tsv_status tsv_verify_accept_sharded(const tsv_verify_args* a, tsv_comm* comm, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(a && comm, "tsv_verify_accept_sharded: NULL argument");
    TSV_TRY(nccl_ready());
    size_t need = 0, slots = 0;
    TSV_TRY(tsv_verify_sharded_workspace_size(a, comm->world, &need));
    TSV_REQUIRE_WS(a->workspace && a->workspace_bytes >= need, "tsv_verify_accept_sharded: workspace too small (%llu < %llu)",
                (unsigned long long)a->workspace_bytes, (unsigned long long)need);
    if (a->B == 0) return TSV_OK;
    TSV_TRY(tsv_verify_workspace_size(a, &slots));
    slots = (slots + 255) & ~static_cast<size_t>(255);
    char* ws = static_cast<char*>(a->workspace);
    tsv_verify_args b = *a;
    b.workspace_bytes = slots;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (a->flags & TSV_VERIFY_SHARD_DENSE) {  // one round: every row of every request
        tsv_shard_tuple* local = reinterpret_cast<tsv_shard_tuple*>(ws + slots);
        tsv_shard_tuple* gathered = local + a->rows_p;
        TSV_TRY(tsv_verify_shard_partial(&b, local, stream));
        const size_t words = static_cast<size_t>(a->rows_p) * sizeof(tsv_shard_tuple) / sizeof(uint64_t);
        TSV_TRY(nccl_status(g_nccl.AllGather(local, gathered, words, ncclUint64, comm->comm, st), "ncclAllGather"));
        return tsv_verify_shard_combine(&b, gathered, comm->world, stream);
    }
    // lazy two rounds: flags -> sum -> race of row m_i only -> max -> emit
    uint64_t* masks = reinterpret_cast<uint64_t*>(ws + slots);
    uint64_t* keys = masks + a->B;
    TSV_TRY(tsv_verify_shard_flags(&b, masks, stream));
    TSV_TRY(nccl_status(g_nccl.AllReduce(masks, masks, static_cast<size_t>(a->B), ncclUint64, ncclSum, comm->comm, st),
                        "ncclAllReduce(sum)"));
    TSV_TRY(tsv_verify_shard_race(&b, masks, keys, stream));
    TSV_TRY(nccl_status(g_nccl.AllReduce(keys, keys, 2 * static_cast<size_t>(a->B), ncclUint64, ncclMax, comm->comm, st),
                        "ncclAllReduce(max)"));
    return tsv_verify_shard_emit(&b, masks, keys, stream);
}

extern "C" tsv_status tsv_allreduce_i64(int64_t* data, size_t count, tsv_comm* comm, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(data && comm, "tsv_allreduce_i64: NULL argument");
    TSV_TRY(nccl_ready());
    return nccl_status(g_nccl.AllReduce(data, data, count, ncclInt64, ncclSum, comm->comm,
                                        static_cast<cudaStream_t>(stream)),
                       "ncclAllReduce");
}

extern "C" tsv_status tsv_goodput_choose_k_sharded(const double* alpha, int32_t alpha_per_request,
                                                   const int32_t* ctx_len, const int32_t* cap, int32_t B,
                                                   int32_t k_max, int32_t policy, tsv_latency_model target,
                                                   tsv_latency_model draft, double pld_cost_ms,
                                                   int64_t kv_free_slots, int32_t* k_out, double* goodput_out,
                                                   int32_t* k_per_request, int64_t* sums_ws, tsv_comm* comm,
                                                   void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(comm && sums_ws, "tsv_goodput_choose_k_sharded: NULL argument");
    TSV_TRY(nccl_ready());
    TSV_TRY(tsv_goodput_partial(alpha, alpha_per_request, ctx_len, cap, B, k_max, sums_ws, stream));
    TSV_TRY(tsv_allreduce_i64(sums_ws, TSV_GP_SUMS(k_max), comm, stream));
    return tsv_goodput_finalize(sums_ws, k_max, policy, target, draft, pld_cost_ms, kv_free_slots, cap, B, k_out,
                                goodput_out, k_per_request, stream);
}

extern "C" tsv_status tsv_update_acceptance_sharded(double* alpha, const int32_t* num_accepted,
                                                    const int32_t* row_offsets, int32_t B, double decay,
                                                    int32_t estimator, int64_t* sums_ws, tsv_comm* comm,
                                                    void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(comm && sums_ws && alpha, "tsv_update_acceptance_sharded: NULL argument");
    TSV_TRY(nccl_ready());
    TSV_TRY(tsv_update_partial(num_accepted, row_offsets, B, estimator, sums_ws, stream));
    TSV_TRY(tsv_allreduce_i64(sums_ws, 2, comm, stream));
    return tsv_update_finalize(alpha, sums_ws, decay, stream);
}

// ------------------------------------------------------------------ diagnostics (tests)
namespace tsv {
__global__ void debug_race_E_kernel(uint32_t m_begin, uint32_t n, float* out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint32_t m = m_begin + t;  // race uniform u = (2m + 1) 2^-24, any word with low bits m
    out[t] = race_E_omu(one_minus_u_race(m));
}

struct DebugKeys {
    uint32_t ks0[10], ks1[10];
};

__global__ void debug_philox_kernel(const uint32_t* ctr, const uint32_t* key, uint32_t n, uint32_t* out,
                                    int32_t race_variant) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint32_t* c = ctr + 4 * t;
    uint4 r;
    if (race_variant) {
        DebugKeys ks;
        for (uint32_t i = 0; i < 10; ++i) {
            ks.ks0[i] = key[0] + i * kPhiloxW0;
            ks.ks1[i] = key[1] + i * kPhiloxW1;
        }
        const RaceCtr rc = race_ctr(c[1], c[2], c[3], key[0], key[1]);
        r = philox_race(rc, c[0], ks);
    } else {
        r = philox4x32_10(c[0], c[1], c[2], c[3], key[0], key[1]);
    }
    out[4 * t + 0] = r.x;
    out[4 * t + 1] = r.y;
    out[4 * t + 2] = r.z;
    out[4 * t + 3] = r.w;
}
}  // namespace tsv

extern "C" tsv_status tsv_debug_race_E(uint32_t m_begin, uint32_t n, float* out, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(out != nullptr, "tsv_debug_race_E: out is NULL");
    TSV_REQUIRE(static_cast<uint64_t>(m_begin) + n <= (1ull << 23), "tsv_debug_race_E: range beyond 2^23");
    TSV_TRY(check_device());
    if (n == 0) return TSV_OK;
    debug_race_E_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(m_begin, n, out);
    TSV_CUDA(cudaGetLastError(), "debug_race_E_kernel launch");
    return TSV_OK;
}

extern "C" tsv_status tsv_debug_philox(const uint32_t* ctr, const uint32_t* key, uint32_t n, uint32_t* out,
                                       int32_t race_variant, void* stream) {
    TSV_TRACE_CALL();
    TSV_REQUIRE(ctr && key && out, "tsv_debug_philox: NULL argument");
    TSV_TRY(check_device());
    if (n == 0) return TSV_OK;
    debug_philox_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(ctr, key, n, out, race_variant);
    TSV_CUDA(cudaGetLastError(), "debug_philox_kernel launch");
    return TSV_OK;
}
