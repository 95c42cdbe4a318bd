// p2p.cuh -- the NVLink peer-memory exchange shared by the vocab-sharded verify (verify.cu) and
// the request-sharded global goodput / acceptance sums (goodput.cu, verify.cu's update CTA).
//
// Every rank owns one symmetric buffer (tsv_p2p_alloc), mapped into every peer (CUDA IPC).
// Each exchanged 32-bit word travels with the call's epoch in one aligned 8-byte word
// {data, epoch} (the "LL" idea: an aligned 8-byte store arrives whole), written with 16-byte
// volatile vector stores into slot [rank][i] of every peer's buffer; the consumer polls its
// own buffer's G slots until every word carries the epoch -- no fence, no grid barrier, no flag
// round trip.  Slots alternate by epoch parity; the epochs live in the buffer header, so
// captured CUDA graphs replay with advancing epochs.  A wait that never completes gives up
// after about two seconds of device time (%globaltimer) and sets TSV_DEVSTATUS_P2P_TIMEOUT.
//
// Slot reuse is safe because a rank writes call e+2's words (same parity as call e) only after
// finishing call e+1, which needed every peer's call-(e+1) words, which each peer pushed after
// reading its call-e words.  All ranks must make the same sequence of exchange calls.
#pragma once

#include "common.cuh"

namespace tsv {

struct P2PView {
    unsigned char* buf[TSV_P2P_MAX_WORLD];  // rank g's symmetric buffer as mapped in this process
    int32_t rank, G, B_max;
};

// header: u32 verify epoch at 0, emit-arrival counter at 4, sums (all-reduce) epoch at 8
constexpr size_t kP2PHdr = 256;
// round 1 slot: 16 B per request {acc, e, own, e}; round 2 slot: 32 B {key lo/hi, fb lo/hi, each with e}
__host__ __device__ constexpr size_t p2p_masks_bytes(int32_t B_max) {
    return 2ull * TSV_P2P_MAX_WORLD * static_cast<size_t>(B_max) * 16ull;
}
constexpr size_t kP2PSumsBytes = 2ull * TSV_P2P_MAX_WORLD * TSV_P2P_MAX_SUMS * 16ull;  // [2][W][n] LL lines
// Fused push (TSV_VERIFY_P2P_FUSED): every race work item (request i, chunk c) of rank `from` pushes its
// chunk key as one LL line into slot [from][c][i] of every peer; [2][W][kP2PMaxChunks][B_max] lines.
constexpr int32_t kP2PMaxChunks = 32;
__host__ __device__ constexpr size_t p2p_ckeys_bytes(int32_t B_max) {
    return 2ull * TSV_P2P_MAX_WORLD * kP2PMaxChunks * static_cast<size_t>(B_max) * 16ull;
}
__host__ __device__ constexpr size_t p2p_buffer_bytes(int32_t B_max) {
    return kP2PHdr + 3ull * p2p_masks_bytes(B_max) + kP2PSumsBytes + p2p_ckeys_bytes(B_max);
}
__device__ __forceinline__ uint32_t* p2p_epoch(const P2PView& V) {
    return reinterpret_cast<uint32_t*>(V.buf[V.rank]);
}
__device__ __forceinline__ uint32_t* p2p_counter(const P2PView& V) {
    return reinterpret_cast<uint32_t*>(V.buf[V.rank]) + 1;
}
__device__ __forceinline__ uint32_t* p2p_sums_epoch(const P2PView& V) {
    return reinterpret_cast<uint32_t*>(V.buf[V.rank]) + 2;
}
__device__ __forceinline__ uint32_t p2p_load_epoch(const P2PView& V) {
    return *reinterpret_cast<volatile uint32_t*>(p2p_epoch(V)) + 1u;  // this call's epoch (E + 1)
}
__device__ __forceinline__ uint4* p2p_masks(const P2PView& V, uint32_t e, int32_t owner, int32_t slot) {
    return reinterpret_cast<uint4*>(V.buf[owner] + kP2PHdr) +
           (static_cast<size_t>(e & 1u) * TSV_P2P_MAX_WORLD + slot) * V.B_max;
}
__device__ __forceinline__ uint4* p2p_keys(const P2PView& V, uint32_t e, int32_t owner, int32_t slot) {
    return reinterpret_cast<uint4*>(V.buf[owner] + kP2PHdr + p2p_masks_bytes(V.B_max)) +
           (static_cast<size_t>(e & 1u) * TSV_P2P_MAX_WORLD + slot) * 2 * V.B_max;
}
__device__ __forceinline__ uint4* p2p_sums(const P2PView& V, uint32_t e, int32_t owner, int32_t from, int32_t j) {
    return reinterpret_cast<uint4*>(V.buf[owner] + kP2PHdr + 3ull * p2p_masks_bytes(V.B_max)) +
           (static_cast<size_t>(e & 1u) * TSV_P2P_MAX_WORLD + from) * TSV_P2P_MAX_SUMS + j;
}
__device__ __forceinline__ uint4* p2p_ckeys(const P2PView& V, uint32_t e, int32_t owner, int32_t from, int32_t c) {
    return reinterpret_cast<uint4*>(V.buf[owner] + kP2PHdr + 3ull * p2p_masks_bytes(V.B_max) + kP2PSumsBytes) +
           ((static_cast<size_t>(e & 1u) * TSV_P2P_MAX_WORLD + from) * kP2PMaxChunks + c) * V.B_max;
}
__device__ __forceinline__ void st_ll(uint4* p, uint4 v) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const uint4* p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#ifndef TSV_P2P_TIMEOUT_NS
#define TSV_P2P_TIMEOUT_NS 2000000000ull
#endif
// Poll one 16-byte LL line until both 8-byte halves carry epoch e (bounded by device time).
__device__ __forceinline__ uint4 ld_ll_wait(const uint4* p, uint32_t e, int32_t* devstatus) {
    uint4 v = ld_ll(p);
    if (v.y == e && v.w == e) return v;
    const unsigned long long t0 = global_ns();
    uint32_t n = 0;
    while (v.y != e || v.w != e) {
        __nanosleep(32);
        if ((++n & 255u) == 0 && global_ns() - t0 > TSV_P2P_TIMEOUT_NS) {  // a peer never arrived
            report(devstatus, TSV_DEVSTATUS_P2P_TIMEOUT);
            break;
        }
        v = ld_ll(p);
    }
    return v;
}

// In-place exact sum over the ranks of v[0..count) int64 (count <= TSV_P2P_MAX_SUMS; v in this
// CTA's shared memory or in global memory owned by this CTA).  CTA-wide: every thread calls.
// Thread j pushes v[j] as two LL words into slot [rank][j] of every peer, then polls its own
// buffer's G slots and writes the sum (int64 addition: exact and order-free, so every rank
// gets the same bits).  Uses the sums epoch (header word 2), advanced at the end.
__device__ __forceinline__ void p2p_allreduce_block(long long* v, int32_t count, const P2PView& V,
                                                    int32_t* devstatus) {
    const uint32_t e = *reinterpret_cast<volatile uint32_t*>(p2p_sums_epoch(V)) + 1u;
    for (int32_t j = threadIdx.x; j < count; j += blockDim.x) {
        const uint64_t x = static_cast<uint64_t>(v[j]);
        for (int32_t g = 0; g < V.G; ++g)
            st_ll(p2p_sums(V, e, g, V.rank, j), make_uint4(static_cast<uint32_t>(x), e, static_cast<uint32_t>(x >> 32), e));
        uint64_t sum = 0;
        for (int32_t g = 0; g < V.G; ++g) {
            const uint4 w = ld_ll_wait(p2p_sums(V, e, V.rank, g, j), e, devstatus);
            sum += (static_cast<uint64_t>(w.z) << 32) | w.x;
        }
        v[j] = static_cast<long long>(sum);
    }
    __syncthreads();  // every thread has read the epoch and finished its slots
    if (threadIdx.x == 0) *p2p_sums_epoch(V) = e;
}

// The same exchange for a pair held by ONE warp (the race grid's update warp): lane j < 2 publishes and
// sums word j; every lane returns with both sums.
__device__ __forceinline__ void p2p_allreduce_warp(long long& a, long long& b, const P2PView& V, int32_t* devstatus) {
    const int lane = threadIdx.x & 31;
    const uint32_t e = *reinterpret_cast<volatile uint32_t*>(p2p_sums_epoch(V)) + 1u;
    if (lane < 2) {
        const uint64_t x = static_cast<uint64_t>(lane == 0 ? a : b);
        for (int32_t g = 0; g < V.G; ++g)
            st_ll(p2p_sums(V, e, g, V.rank, lane), make_uint4(static_cast<uint32_t>(x), e, static_cast<uint32_t>(x >> 32), e));
        uint64_t sum = 0;
        for (int32_t g = 0; g < V.G; ++g) {
            const uint4 w = ld_ll_wait(p2p_sums(V, e, V.rank, g, lane), e, devstatus);
            sum += (static_cast<uint64_t>(w.z) << 32) | w.x;
        }
        if (lane == 0) a = static_cast<long long>(sum);
        else b = static_cast<long long>(sum);
    }
    a = __shfl_sync(0xFFFFFFFFu, a, 0);
    b = __shfl_sync(0xFFFFFFFFu, b, 1);
    __syncwarp();  // both lanes have read the epoch and finished their slots
    if (lane == 0) *p2p_sums_epoch(V) = e;
}

}  // namespace tsv

// The opaque handle of include/tsv.h.
struct tsv_p2p {
    tsv::P2PView view;
};
