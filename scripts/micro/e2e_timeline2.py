"""Wall time of gc_ktruss_analysis(_async) with host / device / no outputs (C4)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import gen
from paper_1708_06866_b200 import Context
u, v = gen.CONFIGS["C4"].generate()
ctx = Context(0, torch.cuda.current_stream())
print("stream", torch.cuda.current_stream())
ctx.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()); ctx.build_csr(); m = ctx.num_edges()
hs = torch.empty(m, dtype=torch.int32).pin_memory(); hm = torch.empty(m, dtype=torch.uint8).pin_memory()
ds = torch.empty(m, dtype=torch.int32, device="cuda"); dm = torch.empty(m, dtype=torch.uint8, device="cuda")
print("pinned", hs.is_pinned(), hm.is_pinned())
for name, f in [("sync host", lambda: ctx.ktruss_analysis(3, hs, hm)),
                ("async host", lambda: ctx.ktruss_analysis_async(3, hs, hm)),
                ("sync dev", lambda: ctx.ktruss_analysis(3, ds, dm)),
                ("async dev", lambda: ctx.ktruss_analysis_async(3, ds, dm))]:
    for i in range(2):
        t0 = time.perf_counter(); f(); t1 = time.perf_counter(); ctx.wait(); t2 = time.perf_counter()
        st = ctx.stats()
        print(f"{name}: call {1e3*(t1-t0):6.1f} ms wait {1e3*(t2-t1):6.1f} ms ktruss_ms {st['ktruss_ms']:.1f}", flush=True)
