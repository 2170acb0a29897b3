"""Exercise every libgc entry point and kernel class on small graphs (stress run; results cross-checked)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen
from paper_1708_06866_b200 import gc

cases = [gen.CONFIGS["C1"].generate(), gen.rmat(12, 16, seed=5), gen.king_grid(40)]
iu, ju = np.triu_indices(300, 1)
cases.append((iu.astype(np.int32), ju.astype(np.int32)))       # K_300: heavy heads
for parts in (0, 2):
    for force in (-1, 1, 2, 3):
        for u, v in cases:
            with gc.Context(0) as c:
                if parts:
                    c.comm_init_loopback(parts)
                c.load_edges(u, v)
                c.set_option(gc.GC_OPT_FORCE_CLASS, force)
                if force == 3:
                    c.set_option(gc.GC_OPT_HUGE_MAX, 16)
                c.build_csr()
                T = c.triangle_count()
                s = c.edge_support()
                T2, s2, mk, ma = c.ktruss_analysis(4)
                c.ktruss(6)
                tau, kmax = c.truss_decomposition()
                tri = c.list_triangles()
                assert T == T2 and np.array_equal(s, s2) and len(tri) == T
print("stress run ok")
