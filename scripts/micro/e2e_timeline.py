"""Host wall-clock timeline of the pipelined e2e loop (C4): where does the time go per call?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import gen
from paper_1708_06866_b200 import Context
u, v = gen.CONFIGS["C4"].generate()
hu = torch.from_numpy(u).pin_memory(); hv = torch.from_numpy(v).pin_memory()
ctx = Context(0, torch.cuda.current_stream())
ctx.load_edges(hu, hv); ctx.build_csr(); m = ctx.num_edges()
hs = torch.empty(m, dtype=torch.int32).pin_memory(); hm = torch.empty(m, dtype=torch.uint8).pin_memory()
for mode in ("sync", "async", "sync-nostage", "async-nostage"):
    ctx.stage_edges(hu, hv)
    for i in range(3):
        t0 = time.perf_counter(); ctx.build_csr(); t1 = time.perf_counter()
        if "nostage" not in mode or i < 2:
            ctx.stage_edges(hu, hv)
        t2 = time.perf_counter()
        if mode.startswith("async"):
            ctx.ktruss_analysis_async(3, hs, hm)
        else:
            ctx.ktruss_analysis(3, hs, hm)
        t3 = time.perf_counter()
        print(f"{mode} step {i}: build {1e3*(t1-t0):6.1f} stage {1e3*(t2-t1):6.1f} analysis {1e3*(t3-t2):6.1f} total {1e3*(t3-t0):6.1f} ms sup {ctx.stats()['support_kernel_ms']:.1f}", flush=True)
    t0 = time.perf_counter(); ctx.wait(); print(f"wait {1e3*(time.perf_counter()-t0):.1f} ms")
    ctx.build_csr()
# raw copy rates
x = torch.empty(hu.numel(), dtype=torch.int32, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); x.copy_(hu, non_blocking=True); torch.cuda.synchronize()
print(f"H2D {hu.numel()*4/1e9:.2f} GB in {1e3*(time.perf_counter()-t0):.1f} ms")
y = torch.empty(m, dtype=torch.int32).pin_memory(); xs = x[:m]
torch.cuda.synchronize(); t0 = time.perf_counter(); y.copy_(xs, non_blocking=True); torch.cuda.synchronize()
print(f"D2H {m*4/1e9:.2f} GB in {1e3*(time.perf_counter()-t0):.1f} ms")
