"""Small support run for compute-sanitizer / bisecting (GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen, oracle
from paper_1708_06866_b200 import gc
s = int(sys.argv[1]) if len(sys.argv) > 1 else 14
u, v = gen.rmat(s, 16, seed=3)
g = oracle.OracleGraph(u, v)
want = g.support()
for sname, opts in [("default", {}), ("force1", {gc.GC_OPT_FORCE_CLASS: 1}), ("force1_nolong", {gc.GC_OPT_FORCE_CLASS: 1, gc.GC_OPT_LONG_SEG: 1 << 30}),
                    ("nolong", {gc.GC_OPT_LONG_SEG: 1 << 30}), ("chunk64", {gc.GC_OPT_TASK_CHUNK: 64})]:
    with gc.Context(0) as c:
        for k, val in opts.items():
            c.set_option(k, val)
        c.load_edges(u, v); c.build_csr()
        sup = c.edge_support()
        st = c.stats()
        print(s, sname, "mismatch", int((sup != want).sum()), "tasks", st["tasks"], flush=True)
