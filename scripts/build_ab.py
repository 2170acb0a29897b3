"""gc_build_csr time on one GPU: the replicated build, and the partitioned
build (GC_OPT_BUILD_PART) under loopback virtual ranks, with each virtual
rank's device time for its share (stats.part_build_ms)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_1708_06866_b200 import gc
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
u, v = gen.CONFIGS[cfg].generate()
du, dv = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
for P in (0, 1, 2, 4, 8):
    ctx = gc.Context(0, torch.cuda.current_stream())
    try:
        if P >= 2:
            ctx.comm_init_loopback(P)
        if P >= 1:
            ctx.set_option(gc.GC_OPT_BUILD_PART, 1)
        ctx.load_edges(du, dv)
        ts, parts = [], None
        for r in range(3):
            ctx.build_csr()
            st = ctx.stats()
            ts.append(st["build_ms"])
            parts = [round(x, 2) for x in st["part_build_ms"][:P]] if P >= 2 else []
        shared = min(ts) - sum(parts)
        print(json.dumps({"config": cfg, "owners": P, "build_ms": round(min(ts), 2), "part_build_ms": parts,
                          "replicated_ms": round(shared, 2) if parts else None,
                          "per_rank_estimate_ms": round(shared + max(parts), 2) if parts else None}), flush=True)
    finally:
        ctx.close()
