"""Diagnostic (not part of the product): per-launch floor of dependent kernels in a CUDA graph.

Times graphs of N back-to-back tiny kernels (1 CTA / 148 CTAs / 296 CTAs; each reads one
value written by its predecessor), launched plainly or with programmatic dependent launch
(griddepcontrol), to separate fixed per-kernel cost from work in the step breakdown.
"""
import torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <cuda_runtime.h>
__global__ void chain(int* x, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) x[0] = x[0] + 1;
}
void launch(torch::Tensor x, int grid, int pdl, int n) {
    auto st = at::cuda::getCurrentCUDAStream().stream();
    for (int i = 0; i < n; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr; cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, chain, x.data_ptr<int>(), pdl);
    }
}
"""
mod = load_inline("diag_launch", cpp_sources="void launch(torch::Tensor x, int grid, int pdl, int n);",
                  cuda_sources="#include <ATen/cuda/CUDAContext.h>\n" + src, functions=["launch"],
                  extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"], verbose=False)
x = torch.zeros(1, dtype=torch.int32, device="cuda")
N = 64
for grid in (1, 148, 296, 592):
    for pdl in (0, 1):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            mod.launch(x, grid, pdl, 1)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                mod.launch(x, grid, pdl, N)
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"grid {grid:4d} pdl {pdl}: {e0.elapsed_time(e1) / (20 * N) * 1e3:6.2f} us per dependent launch")
