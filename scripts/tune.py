"""Time TC/support at one config over option settings: python scripts/tune.py C4 'opt=val,opt=val' ..."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_1708_06866_b200 import gc
cfg = sys.argv[1]
u, v = gen.CONFIGS[cfg].generate()
du, dv = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
ctx = gc.Context(0, torch.cuda.current_stream())
ctx.load_edges(du, dv)
ctx.build_csr()
out = torch.empty(ctx.num_edges(), dtype=torch.int32, device="cuda")
print("stats", {k: ctx.stats()[k] for k in ("n", "m", "wedges", "max_out_degree", "tasks", "aux")}, flush=True)
for spec in sys.argv[2:]:
    opts = {}
    for kv in filter(None, spec.split(",")):
        k, val = kv.split("=")
        opts[getattr(gc, "GC_OPT_" + k.upper())] = int(val)
    for k, val in opts.items():
        ctx.set_option(k, val)
    tcs, sps = [], []
    for r in range(3):
        ctx.triangle_count(); tcs.append(ctx.stats()["tc_kernel_ms"])
        ctx.edge_support(out); sps.append(ctx.stats()["support_kernel_ms"])
    print(f"{spec:40s} tc {min(tcs):8.2f} ms  support {min(sps):8.2f} ms", flush=True)
