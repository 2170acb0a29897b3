"""Micro-benchmark: the libgc-style grid-stride 4-byte scatter kernel under different index orders."""
import torch
from torch.utils.cpp_extension import load_inline
src = r'''
#include <torch/extension.h>
__global__ void k(const int* __restrict__ idx, const int* __restrict__ vals, long m, int* __restrict__ out) {
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < m; p += (long)gridDim.x * blockDim.x)
        out[idx[p]] = vals[p];
}
void scat(torch::Tensor idx, torch::Tensor vals, torch::Tensor out, int grid) {
    k<<<grid, 256>>>(idx.data_ptr<int>(), vals.data_ptr<int>(), idx.numel(), out.data_ptr<int>());
}
'''
mod = load_inline("scat_mod", cpp_sources="void scat(torch::Tensor idx, torch::Tensor vals, torch::Tensor out, int grid);",
                  cuda_sources=src, functions=["scat"], extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a"])
m = 260_381_325
g = torch.Generator(device="cuda").manual_seed(0)
val = torch.randint(0, 1 << 30, (m,), device="cuda", dtype=torch.int32)
out = torch.empty(m, device="cuda", dtype=torch.int32)
perm = torch.randperm(m, device="cuda", generator=g).to(torch.int32)
def t(idx, name, grid, reps=5):
    mod.scat(idx, val, out, grid); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): mod.scat(idx, val, out, grid)
    b.record(); torch.cuda.synchronize()
    print(f"{name:40s} grid {grid:7d} {a.elapsed_time(b)/reps:7.3f} ms", flush=True)
for grid in (148 * 16, (m + 255) // 256):
    t(torch.arange(m, device="cuda", dtype=torch.int32), "identity", grid)
    t(perm, "random permutation", grid)
    for bits in (20, 12):
        order = torch.argsort(perm >> bits, stable=True)
        t(perm[order].contiguous(), f"sorted on id >> {bits}", grid)
