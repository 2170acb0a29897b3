"""Drive one config through build + TC + support (+ktruss) N times (for ncu / timing)."""
import argparse
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_1708_06866_b200 import Context

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--reps", type=int, default=2)
p.add_argument("--what", default="tc,support")
p.add_argument("--chunk", type=int, default=0)
p.add_argument("--k", type=int, default=3, help="k of the analysis / ktruss calls")
p.add_argument("--opt", action="append", default=[], help="OPTION_ID=VALUE (gc_set_option)")
a = p.parse_args()
u, v = gen.CONFIGS[a.config].generate()
ctx = Context(0, torch.cuda.current_stream())
if a.chunk:
    ctx.set_option(2, a.chunk)
for o in a.opt:
    oid, oval = o.split("=")
    ctx.set_option(int(oid), int(oval))
ctx.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
for r in range(a.reps):
    ctx.build_csr()
    if "tc" in a.what:
        T = ctx.triangle_count()
    if "support" in a.what:
        ctx.edge_support(torch.empty(ctx.num_edges(), dtype=torch.int32, device="cuda"))
    if "analysis" in a.what:
        ctx.ktruss_analysis(a.k, torch.empty(ctx.num_edges(), dtype=torch.int32, device="cuda"),
                            torch.empty(ctx.num_edges(), dtype=torch.uint8, device="cuda"))
    if "ktruss" in a.what:
        ctx.ktruss(a.k, torch.empty(ctx.num_edges(), dtype=torch.uint8, device="cuda"))
    st = ctx.stats()
    print({k: st[k] for k in ["build_ms", "tc_kernel_ms", "support_kernel_ms", "ktruss_ms", "peel_ms", "tasks"]}, flush=True)
