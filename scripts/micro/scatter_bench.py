"""Micro-benchmark: 4-byte scatter out[idx[p]] = val[p] under different index orders (m = C4's 2.6e8)."""
import torch
m = 260_381_325
g = torch.Generator(device="cuda").manual_seed(0)
val = torch.randint(0, 1 << 30, (m,), device="cuda", dtype=torch.int32)
out = torch.empty(m, device="cuda", dtype=torch.int32)
perm = torch.randperm(m, device="cuda", generator=g)
def t(idx, name, reps=5):
    out.index_copy_(0, idx, val); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): out.index_copy_(0, idx, val)
    b.record(); torch.cuda.synchronize()
    print(f"{name:40s} {a.elapsed_time(b)/reps:7.3f} ms", flush=True)
t(torch.arange(m, device="cuda"), "identity")
t(perm, "random permutation")
for bits in (20, 16, 12, 8):
    key = perm >> bits
    order = torch.argsort(key, stable=True)
    t(perm[order], f"sorted on id >> {bits} (window {4 << bits >> 10} KB)")
