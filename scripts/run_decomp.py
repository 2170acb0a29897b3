"""Time gc_truss_decomposition (and ktruss at a few k) on one config."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_1708_06866_b200 import gc

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--ks", default="")
p.add_argument("--part", type=int, default=0)
p.add_argument("--loop", type=int, default=0)
p.add_argument("--tc", type=int, default=0)
p.add_argument("--compact", type=int, default=-1)
p.add_argument("--group", type=int, default=-1)
p.add_argument("--heavy", type=int, default=-1)
p.add_argument("--no-decomp", action="store_true")
a = p.parse_args()
t0 = time.time()
u, v = gen.CONFIGS[a.config].generate()
print(f"gen {time.time()-t0:.1f}s nnz={u.size}", flush=True)
ctx = gc.Context(0, torch.cuda.current_stream())
if a.loop:
    ctx.comm_init_loopback(a.loop)
if a.group >= 0:
    ctx.set_option(gc.GC_OPT_GROUP_PEEL, a.group)
if a.heavy >= 0:
    ctx.set_option(gc.GC_OPT_GROUP_HEAVY, a.heavy)
if a.compact >= 0:
    ctx.set_option(gc.GC_OPT_COMPACT, a.compact)
if a.part:
    ctx.set_option(gc.GC_OPT_PEEL_PART, 1)
ctx.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
ctx.build_csr()
m = ctx.num_edges()
st = ctx.stats()
print(f"n={ctx.num_vertices()} m={m} build {st['build_ms']:.1f} ms", flush=True)
if a.tc:
    for r in range(a.tc):
        T = ctx.triangle_count()
        sup = torch.empty(m, dtype=torch.int32, device="cuda")
        ctx.edge_support(sup)
        st = ctx.stats()
        print(f"T={T} tc {st['tc_kernel_ms']:.1f} ms support {st['support_kernel_ms']:.1f} ms wedges={st['wedges']} "
              f"maxdeg={st['max_degree']} max_out={st['max_out_degree']} tasks={list(st['tasks'])}", flush=True)
    print(f"mem peak {torch.cuda.mem_get_info()}", flush=True)
for k in [int(x) for x in a.ks.split(",") if x]:
    mask = torch.empty(m, dtype=torch.uint8, device="cuda")
    _, alive = ctx.ktruss(k, mask)
    st = ctx.stats()
    print(f"ktruss({k}): {alive} edges, {st['ktruss_ms']:.1f} ms (peel {st['peel_ms']:.1f} ms, {st['peel_rounds']} rounds)", flush=True)
if a.no_decomp:
    sys.exit(0)
tau = torch.empty(m, dtype=torch.int32, device="cuda")
t0 = time.time()
_, kmax = ctx.truss_decomposition(tau)
st = ctx.stats()
print(f"decomposition: kmax={kmax} {st['decomp_ms']:.1f} ms (peel {st['peel_ms']:.1f} ms, {st['peel_rounds']} rounds, {st['compactions']} compactions) wall {time.time()-t0:.2f}s "
      f"kernel {st['peel_kernel_ms']:.1f} scan {st['scan_ms']:.1f} compact {st['compact_ms']:.1f} ms", flush=True)
