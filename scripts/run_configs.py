"""Per-config report (VERDICT r1 "Reporting"): one JSON line per config C1..C5
and a markdown table.

GPU side (libgc through its C ABI, one B200): gc_build_csr, the triangle
count pass, the support pass, k-truss k = 3..6 (gc_ktruss_analysis) and the
full decomposition, device times from the library's CUDA events (best of
--reps), plus device memory in use after the run (the library pool keeps
every block it allocated, so this is the peak) and the processor fields the
paper reports (GPU / CPU model, core counts).

Oracle side (oracle/, test infrastructure): canonicalise + adjacency, O-3
support and O-4 triangle count at 1 thread and at all host cores, for the
configs where that takes minutes at most (C1-C3; C4/C5 quote the full runs
recorded by scripts/make_golden.py in tests/golden/c?_expected.json).

    python scripts/run_configs.py [--configs C1,C2,C3,C4,C5] [--oracle] [--out profiles/round2]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def gpu_side(name, reps):
    import torch
    import gen
    from paper_1708_06866_b200 import gc
    cfg = gen.CONFIGS[name]
    u, v = cfg.generate()
    nnz = int(u.size)
    free0, total = torch.cuda.mem_get_info()
    ctx = gc.Context(0, torch.cuda.current_stream())
    out = {"config": name, "desc": cfg.desc, "nnz": nnz}
    try:
        ctx.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
        del u, v
        best = {}

        def keep(key, val):
            best[key] = min(best.get(key, float("inf")), val)

        for r in range(reps):
            ctx.build_csr()
            keep("build_ms", ctx.stats()["build_ms"])
        m, n = ctx.num_edges(), ctx.num_vertices()
        sup = torch.empty(m, dtype=torch.int32, device="cuda")
        mask = torch.empty(m, dtype=torch.uint8, device="cuda")
        tau = torch.empty(m, dtype=torch.int32, device="cuda")
        for r in range(reps):
            T = ctx.triangle_count()
            keep("tc_kernel_ms", ctx.stats()["tc_kernel_ms"])
            ctx.edge_support(sup)
            keep("support_kernel_ms", ctx.stats()["support_kernel_ms"])
        kt = {}
        for k in (3, 4, 5, 6):
            for r in range(reps):
                _, _, _, ma = ctx.ktruss_analysis(k, sup, mask)
                st = ctx.stats()
                kt.setdefault(str(k), {"edges": ma, "ms": float("inf"), "rounds": st["peel_rounds"]})
                kt[str(k)]["ms"] = min(kt[str(k)]["ms"], st["ktruss_ms"])
        dreps = 1 if m > 50_000_000 else reps
        for r in range(dreps):
            _, kmax = ctx.truss_decomposition(tau)
            st = ctx.stats()
            keep("decomposition_ms", st["decomp_ms"])
        st = ctx.stats()
        free1, _ = torch.cuda.mem_get_info()
        out.update(n=n, m=m, triangles=T, kmax=kmax, decomposition_rounds=st["peel_rounds"], ktruss=kt,
                   **{k: round(v, 3) for k, v in best.items()},
                   tc_rate_edges_per_s=m / (best["tc_kernel_ms"] / 1e3),
                   support_rate_edges_per_s=m / (best["support_kernel_ms"] / 1e3),
                   device_memory_gb=round((free0 - free1) / 1e9, 2),
                   work={k: st[k] for k in ("wedges", "q_out", "q_in", "max_out_degree", "max_degree")})
    finally:
        ctx.close()
    props = torch.cuda.get_device_properties(0)
    out["processor"] = {"gpu": props.name, "sms": props.multi_processor_count,
                        "gpu_memory_gb": round(total / 1e9, 1), "cpu": cpu_model(), "cores": os.cpu_count()}
    return out


def oracle_side(name):
    import gen
    import oracle
    cfg = gen.CONFIGS[name]
    u, v = cfg.generate()
    res = {}
    for threads in (1, os.cpu_count() or 1):
        t0 = time.perf_counter()
        g = oracle.OracleGraph(u, v, nthreads=threads)
        t1 = time.perf_counter()
        g.support()
        t2 = time.perf_counter()
        g.triangle_count()
        t3 = time.perf_counter()
        res[str(threads)] = {"canonicalize_adjacency_s": round(t1 - t0, 3), "support_s": round(t2 - t1, 3),
                             "triangle_count_s": round(t3 - t2, 3),
                             "tc_support_edges_per_s": g.m / (t3 - t0)}
    return {"threads": res, "cpu": cpu_model(), "where": "this run's host"}


def golden_times(name):
    p = os.path.join(ROOT, "tests", "golden", f"{name.lower()}_expected.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return {**d.get("oracle_times", {}), "where": "scripts/make_golden.py (build container)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "round2"))
    ap.add_argument("--render", help="only re-render configs.md from this configs.jsonl")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    if a.render:
        write_md([json.loads(ln) for ln in open(a.render) if ln.strip()], a.out)
        return
    lines = []
    for name in a.configs.split(","):
        d = gpu_side(name, a.reps)
        if a.oracle and name in ("C1", "C2", "C3"):
            d["oracle"] = oracle_side(name)
        elif golden_times(name):
            d["oracle"] = golden_times(name)
        print(json.dumps(d), flush=True)
        lines.append(d)
    with open(os.path.join(a.out, "configs.jsonl"), "w") as f:
        for d in lines:
            f.write(json.dumps(d) + "\n")
    write_md(lines, a.out)


def write_md(lines, out):
    with open(os.path.join(out, "configs.md"), "w") as f:
        f.write("# Per-config results (scripts/run_configs.py)\n\n")
        f.write("Device times: best of the runs, CUDA events inside libgc. Rates: m / kernel time.\n\n")
        f.write("| config | n | m | T | build ms | TC ms | TC edges/s | support ms | k=3..6 ms | decomposition | mem GB |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|---|\n")
        for d in lines:
            ks = " / ".join(f"{d['ktruss'][k]['ms']:.1f}" for k in ("3", "4", "5", "6"))
            f.write(f"| {d['config']} | {d['n']:,} | {d['m']:,} | {d['triangles']:,} | {d['build_ms']:.1f} | "
                    f"{d['tc_kernel_ms']:.2f} | {d['tc_rate_edges_per_s']:.3g} | {d['support_kernel_ms']:.2f} | {ks} | "
                    f"kmax {d['kmax']}, {d['decomposition_rounds']} rounds, {d['decomposition_ms']:.0f} ms | "
                    f"{d['device_memory_gb']} |\n")
        f.write("\nOracle (CPU) per config:\n\n| config | where | threads | canon+adj s | support s | TC s | TC+support edges/s |\n|---|---|---|---|---|---|---|\n")
        for d in lines:
            o = d.get("oracle")
            if not o:
                continue
            if isinstance(o.get("threads"), dict):
                for t, r in o["threads"].items():
                    f.write(f"| {d['config']} | {o['where']} ({o['cpu']}) | {t} | {r['canonicalize_adjacency_s']} | "
                            f"{r['support_s']} | {r['triangle_count_s']} | {r['tc_support_edges_per_s']:.3g} |\n")
            else:
                full = o.get("canonicalize_adjacency_s", 0) + o.get("support_s", 0) + o.get("triangle_count_s", 0)
                f.write(f"| {d['config']} | {o['where']} ({o.get('cpu')}) | {o.get('threads')} | "
                        f"{o.get('canonicalize_adjacency_s')} | {o.get('support_s')} | {o.get('triangle_count_s')} | "
                        f"{d['m'] / full:.3g} |\n")
                if o.get("truss_sequential_s"):
                    f.write(f"| {d['config']} | O-7 decomposition, 1 thread | 1 | | | | {o['truss_sequential_s']} s |\n")
        f.write("\nProcessor: " + json.dumps(lines[0]["processor"]) + "\n")


if __name__ == "__main__":
    main()
