"""Partitioned (multi-GPU) code paths timed on ONE GPU through loopback
virtual ranks (gc_comm_init_loopback): the P owners run one after another on
this device, so times add up over the ranks; what this measures is the
balance of the 1D cost cut (per-rank intersection time, stats.part_ms) and
the partitioned peeler's total work against the single-rank peeler.

    python scripts/loopback_scaling.py [C4] [--parts 0,1,2,4,8] [--decomp]
P = 0: the single-rank peeler; P = 1: the partitioned peeler on one owner
(GC_OPT_PEEL_PART); P >= 2: loopback virtual ranks.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_1708_06866_b200 import gc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="C4")
ap.add_argument("--parts", default="0,1,2,4,8")
ap.add_argument("--decomp", action="store_true")
a = ap.parse_args()
u, v = gen.CONFIGS[a.config].generate()
du, dv = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
ref = None
for P in [int(x) for x in a.parts.split(",")]:
    ctx = gc.Context(0, torch.cuda.current_stream())
    try:
        if P >= 2:
            ctx.comm_init_loopback(P)
        elif P == 1:
            ctx.set_option(gc.GC_OPT_PEEL_PART, 1)
        ctx.load_edges(du, dv)
        ctx.build_csr()
        m = ctx.num_edges()
        sup = torch.empty(m, dtype=torch.int32, device="cuda")
        mask = torch.empty(m, dtype=torch.uint8, device="cuda")
        ctx.edge_support(sup)
        ctx.edge_support(sup)
        st = ctx.stats()
        parts = [x for x in st["part_ms"][: max(P, 1)] if x > 0] if P >= 2 else []
        out = {"config": a.config, "P": P, "support_ms": st["support_kernel_ms"],
               "part_ms": parts,
               "part_max_over_mean": (max(parts) / (sum(parts) / len(parts))) if parts else None}
        ctx.triangle_count()                     # first call: per-context launch set-up
        ctx.triangle_count()
        out["tc_ms"] = ctx.stats()["tc_kernel_ms"]
        tcp = [x for x in ctx.stats()["part_ms"][: max(P, 1)] if x > 0] if P >= 2 else []
        out["tc_part_ms"] = tcp
        out["tc_part_max_over_mean"] = (max(tcp) / (sum(tcp) / len(tcp))) if tcp else None
        for k in (4, 6):
            ctx.ktruss_analysis(k, sup, mask)
            st = ctx.stats()
            out[f"ktruss{k}_ms"] = st["ktruss_ms"]
            out[f"ktruss{k}_peel_ms"] = st["peel_ms"]
            out[f"ktruss{k}_rounds"] = st["peel_rounds"]
            out[f"ktruss{k}_edges"] = int(mask.sum().item())
        if a.decomp:
            tau = torch.empty(m, dtype=torch.int32, device="cuda")
            _, kmax = ctx.truss_decomposition(tau)
            st = ctx.stats()
            out.update(decomposition_ms=st["decomp_ms"], kmax=kmax, decomposition_rounds=st["peel_rounds"])
            h = int(torch.sum(tau.to(torch.int64) * torch.arange(1, m + 1, device="cuda", dtype=torch.int64) % 1000003).item())
            out["tau_check"] = h
            if ref is None:
                ref = h
            out["tau_equal_to_first"] = h == ref
        print(json.dumps(out), flush=True)
    finally:
        ctx.close()
