"""Bisect support mismatches over kernel options (GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, oracle
from paper_1708_06866_b200 import gc
cases = [("s16", gen.rmat(16, 16, seed=3)), ("s18", gen.rmat(18, 16, seed=3)), ("C3", gen.CONFIGS["C3"].generate())]
settings = [("default", {}), ("nolong", {gc.GC_OPT_LONG_SEG: 1 << 30}), ("long1", {gc.GC_OPT_LONG_SEG: 1}),
            ("hash", {gc.GC_OPT_BLOCK_BITMAP: 0}), ("cls2", {gc.GC_OPT_FORCE_CLASS: 2}),
            ("cls3", {gc.GC_OPT_FORCE_CLASS: 3}), ("chunk_big", {gc.GC_OPT_TASK_CHUNK: 1 << 28})]
for name, (u, v) in cases:
    g = oracle.OracleGraph(u, v)
    want = g.support()
    T = g.triangle_count()
    for sname, opts in settings:
        with gc.Context(0) as c:
            for k, val in opts.items():
                c.set_option(k, val)
            c.load_edges(u, v); c.build_csr()
            t = c.triangle_count(); s = c.edge_support()
            bad = np.flatnonzero(s != want)
            print(name, sname, "T ok" if t == T else f"T BAD {t} vs {T}", "mismatch", bad.size,
                  "diff sum", int(s.astype(np.int64).sum() - want.astype(np.int64).sum()),
                  "first", [(int(g.cu[i]), int(g.cv[i]), int(s[i]), int(want[i])) for i in bad[:3]], flush=True)
