"""k-truss and decomposition times on a config over peeler option settings:
python scripts/peel_ab.py C4 'sort_front=0' 'sort_front=1000000' ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_1708_06866_b200 import gc
cfg = sys.argv[1]
u, v = gen.CONFIGS[cfg].generate()
ctx = gc.Context(0, torch.cuda.current_stream())
ctx.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
ctx.build_csr()
m = ctx.num_edges()
sup = torch.empty(m, dtype=torch.int32, device="cuda")
mask = torch.empty(m, dtype=torch.uint8, device="cuda")
tau = torch.empty(m, dtype=torch.int32, device="cuda")
ctx.ktruss_analysis(4, sup, mask)
for spec in sys.argv[2:]:
    for kv in filter(None, spec.split(",")):
        k, val = kv.split("=")
        ctx.set_option(getattr(gc, "GC_OPT_" + k.upper()), int(val))
    res = []
    for k in (4, 6):
        best = 1e9
        for r in range(3):
            ctx.ktruss_analysis(k, sup, mask)
            best = min(best, ctx.stats()["peel_ms"])
        res.append(f"k{k} peel {best:7.2f} ms")
    ctx.truss_decomposition(tau)
    st = ctx.stats()
    print(f"{spec:28s} {'  '.join(res)}  decomposition {st['decomp_ms']:8.1f} ms (kernel {st['peel_kernel_ms']:.1f})",
          flush=True)
