"""Diagnostic: the CPU oracle's O-3 merge cost model per config (sum over edges
of |N(a)| + |N(b)|, or min * log2(max) when one list is >= 32x longer), to
estimate full-oracle run times from a measured config."""
import sys, os, math
sys.path.insert(0, os.getcwd())
import torch, gen
from paper_1708_06866_b200 import Context
for cfg in sys.argv[1:]:
    u, v = gen.CONFIGS[cfg].generate()
    c = Context(0, torch.cuda.current_stream())
    c.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()); del u, v
    c.build_csr()
    cu, cv = c.get_edges()
    c.close()
    cu = torch.from_numpy(cu).cuda().long(); cv = torch.from_numpy(cv).cuda().long()
    n = int(max(cu.max(), cv.max())) + 1
    deg = (torch.bincount(cu, minlength=n) + torch.bincount(cv, minlength=n)).double()
    da, db = deg[cu], deg[cv]
    lo, hi = torch.minimum(da, db), torch.maximum(da, db)
    merge = float((da + db).sum())
    gal = torch.where(hi >= 32 * lo, lo * torch.log2(hi + 1), da + db)
    print(cfg, "m", cu.numel(), "merge", f"{merge:.3e}", "gallop-model", f"{float(gal.sum()):.3e}", flush=True)
