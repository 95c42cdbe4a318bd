"""Diagnostic (not part of the product): achievable read bandwidth for verify's access pattern.

Streams exactly the rows one verify launch reads on config 2 (row m_i of p for every
request, plus row m_i of q on a rejection) with a trivial sum, under several launch
shapes, and a contiguous copy for reference.  Prints GB/s.  Run on the GPU box:
    python scripts/diag_bw.py
"""
import os
import sys

import torch
from torch.utils.cpp_extension import load_inline

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

src = r"""
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
// items: (row pointer index, chunk); each warp streams one chunk of `chunk` columns per item
__global__ void stream_items(const float* const* rows, int n_rows, int V, int chunk, int unroll, float* out) {
    const int lane = threadIdx.x & 31;
    const long long warp = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * (blockDim.x / 32);
    const int n_chunks = (V + chunk - 1) / chunk;
    const long long n_items = (long long)n_rows * n_chunks;
    float acc = 0.f;
    for (long long it = warp; it < n_items; it += nw) {
        const int r = (int)(it / n_chunks), c = (int)(it % n_chunks);
        const float4* p = reinterpret_cast<const float4*>(rows[r] + (long long)c * chunk);
        const int nq = min(chunk, V - c * chunk) / 4;
        for (int f = lane; f < nq; f += 32 * 4) {
            float4 a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = (f + 32 * u < nq) ? ldg_stream(p + f + 32 * u) : make_float4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += a[u].x + a[u].y + a[u].z + a[u].w;
        }
    }
    if (acc == 12345.f) out[0] = acc;
}
__device__ __forceinline__ uint32_t mulhilo(uint32_t a, uint32_t m, uint32_t& hi) {
    const unsigned long long p = (unsigned long long)a * m; hi = (uint32_t)(p >> 32); return (uint32_t)p;
}
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, hi1;
        const uint32_t lo0 = mulhilo(c0, 0xD2511F53u, hi0);
        const uint32_t lo1 = mulhilo(c2, 0xCD9E8D57u, hi1);
        c0 = hi1 ^ c1 ^ (k0 + r * 0x9E3779B9u); c1 = lo1; c2 = hi0 ^ c3 ^ (k1 + r * 0xBB67AE85u); c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}
template <int ALU>
__global__ void stream_alu(const float* const* rows, int n_rows, int V, int chunk, float* out, uint32_t k0, uint32_t k1) {
    const int lane = threadIdx.x & 31;
    const long long warp = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * (blockDim.x / 32);
    const int n_chunks = (V + chunk - 1) / chunk;
    const long long n_items = (long long)n_rows * n_chunks;
    float acc = 0.f; uint32_t x = 0;
    for (long long it = warp; it < n_items; it += nw) {
        const int r = (int)(it / n_chunks), c = (int)(it % n_chunks);
        const float4* p = reinterpret_cast<const float4*>(rows[r] + (long long)c * chunk);
        const int nq = min(chunk, V - c * chunk) / 4;
        for (int f = lane; f < nq; f += 32 * 4) {
            float4 a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = (f + 32 * u < nq) ? ldg_stream(p + f + 32 * u) : make_float4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (ALU) {
                    const uint4 w = philox(c * chunk / 4 + f + 32 * u, 0x10000u, r, 7, k0, k1);
                    const float t = __uint_as_float((w.x & 0x7FFFFF) ^ 0x3FFFFFFF);
                    acc += (a[u].x > t * 1e-3f) + (a[u].y > __uint_as_float((w.y & 0x7FFFFF) ^ 0x3FFFFFFF) * 1e-3f);
                    x ^= w.z ^ w.w;
                } else {
                    acc += a[u].x + a[u].y + a[u].z + a[u].w;
                }
            }
        }
    }
    if (acc == 12345.f || x == 0x12345678u) out[0] = acc + x;
}
void launch(torch::Tensor rows, int n_rows, int V, int chunk, int grid, int block, torch::Tensor out) {
    stream_items<<<grid, block>>>((const float* const*)rows.data_ptr(), n_rows, V, chunk, 4, out.data_ptr<float>());
}
void launch_alu(torch::Tensor rows, int n_rows, int V, int chunk, int grid, int block, torch::Tensor out) {
    stream_alu<1><<<grid, block>>>((const float* const*)rows.data_ptr(), n_rows, V, chunk, out.data_ptr<float>(), 123u, 456u);
}
"""
cpp = "void launch(torch::Tensor rows, int n_rows, int V, int chunk, int grid, int block, torch::Tensor out);\nvoid launch_alu(torch::Tensor rows, int n_rows, int V, int chunk, int grid, int block, torch::Tensor out);"
mod = load_inline("diag_bw", cpp_sources=cpp, cuda_sources=src, functions=["launch", "launch_alu"],
                  extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"], verbose=False)

import synth  # noqa: E402
from paper_2406_14066_b200 import tsv  # noqa: E402

dev = torch.device("cuda")
sets = []
for s in range(4):
    vb = synth.make_verify_batch(B=256, V=32000, k_max=8, lam=0.7, seed=11 + s, device=dev)
    na, _ = tsv.tsv_verify_accept(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 5, 0, 8)
    torch.cuda.synchronize()
    m = na.long()
    k = vb.k.long()
    ro = vb.row_offsets.long()
    prow = ro[:-1] + m
    ptrs = [vb.p.data_ptr() + int(r) * vb.p.stride(0) * 4 for r in prow.tolist()]
    qb = ro[:-1] - torch.arange(256, device=dev)
    for i in range(256):
        if int(m[i]) < int(k[i]):
            ptrs.append(vb.q.data_ptr() + int(qb[i] + m[i]) * vb.q.stride(0) * 4)
    sets.append((vb, torch.tensor(ptrs, dtype=torch.int64, device=dev), len(ptrs)))
nbytes = sum(n for _, _, n in sets) / len(sets) * 32000 * 4
out = torch.zeros(1, device=dev)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
print(f"rows per step ~{sum(n for *_, n in sets) / 4:.0f}, bytes {nbytes / 1e6:.1f} MB, SMs {sms}")


def time_it(fn, reps=50):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(reps):
        fn(r)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for chunk in (1024, 2048, 4096):
    for block, per_sm in ((256, 3), (256, 4), (256, 8)):
        grid = sms * per_sm
        us = time_it(lambda r: mod.launch(sets[r % 4][1], sets[r % 4][2], 32000, chunk, grid, block, out))
        us2 = time_it(lambda r: mod.launch_alu(sets[r % 4][1], sets[r % 4][2], 32000, chunk, grid, block, out))
        print(f"chunk {chunk:6d} block {block} grid {grid:5d}: stream {us:7.2f} us  {nbytes / us / 1e3:6.0f} GB/s | +philox {us2:7.2f} us  {nbytes / us2 / 1e3:6.0f} GB/s")

x = torch.empty(int(nbytes) // 4, device=dev)
y = torch.empty_like(x)
us = time_it(lambda r: y.copy_(x))
print(f"contiguous copy of {nbytes / 1e6:.0f} MB (read+write): {us:.2f} us, {2 * nbytes / us / 1e3:.0f} GB/s")
