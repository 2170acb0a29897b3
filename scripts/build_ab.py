"""Time gc_build_csr under both build algorithms (GC_OPT_BUILD 0 / 1) on a config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_1708_06866_b200 import gc
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
u, v = gen.CONFIGS[cfg].generate()
ctx = gc.Context(0, torch.cuda.current_stream())
ctx.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
for mode in (0, 1, 0, 1):
    ctx.set_option(gc.GC_OPT_BUILD, mode)
    ts = []
    for r in range(4):
        ctx.build_csr()
        ts.append(ctx.stats()["build_ms"])
    print(f"{cfg} build mode {mode}: min {min(ts):.2f} ms  all {[round(t, 2) for t in ts]}", flush=True)
