"""Diagnostic: per-head work distribution of the block class (d+ in (128, 4096]) at C4."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np, gen
from paper_1708_06866_b200 import Context
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
u, v = gen.CONFIGS[cfg].generate()
c = Context(0, torch.cuda.current_stream())
c.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()); del u, v
c.build_csr()
print("aux", c.stats()["aux"])
cu, cv = c.get_edges()
c.close()
cu = torch.from_numpy(cu).cuda().long(); cv = torch.from_numpy(cv).cuda().long()
n = int(max(cu.max(), cv.max())) + 1
deg = torch.bincount(cu, minlength=n) + torch.bincount(cv, minlength=n)
key = deg * n + torch.arange(n, device="cuda")
order = torch.argsort(key)
rank = torch.empty_like(order); rank[order] = torch.arange(n, device="cuda")
ru, rv = rank[cu], rank[cv]
t = torch.minimum(ru, rv); h = torch.maximum(ru, rv)
del cu, cv, ru, rv
k = t * n + h
k, _ = torch.sort(k)
t = k // n; h = k % n
dplus = torch.bincount(t, minlength=n)
ptr = torch.zeros(n + 1, dtype=torch.long, device="cuda"); ptr[1:] = torch.cumsum(dplus, 0)
pos = torch.arange(t.numel(), device="cuda")
suffix = ptr[t + 1] - pos - 1          # suffix length of in-edge t->h in N+(t) past h
W = torch.zeros(n, dtype=torch.long, device="cuda").index_add_(0, h, suffix)   # wedges streamed for head h
din = torch.bincount(h, minlength=n)
sel = (dplus > 128) & (dplus <= 4096) & (W > 0)
print("class-2 heads", int(sel.sum()), "work", int(W[sel].sum()), "of total", int(W.sum()))
Ws = W[sel].float(); Ds = dplus[sel].float()
for lo, hi in [(0, 1e3), (1e3, 1e4), (1e4, 1e5), (1e5, 1e6), (1e6, 1e7), (1e7, 1e12)]:
    m_ = (Ws >= lo) & (Ws < hi)
    print(f"W in [{lo:.0e},{hi:.0e}): heads {int(m_.sum())}, work {float(Ws[m_].sum()):.3e}, d+ sum {float(Ds[m_].sum()):.3e}")
span = torch.zeros(n, dtype=torch.long, device="cuda")
last = ptr[1:] - 1
span = torch.where(dplus > 0, h[last.clamp(min=0)] - torch.arange(n, device="cuda"), torch.zeros_like(span))
sp = span[sel].float()
for lo, hi in [(0, 2**17), (2**17, 2**18), (2**18, 2**20), (2**20, 2**30)]:
    m_ = (sp >= lo) & (sp < hi)
    print(f"span in [{lo},{hi}): heads {int(m_.sum())}, work {float(Ws[m_].sum()):.3e}")
# class-3 composition (d+ > 4096, or span > 2^18 with d+ > 2048)
c3 = (W > 0) & ((dplus > 4096) | ((span > 2**18) & (dplus > 2048)))
print("class-3 heads", int(c3.sum()), "work", int(W[c3].sum()))
for name, msk in [("2048<d<=4096, span>2^18", (dplus > 2048) & (dplus <= 4096) & (span > 2**18)),
                  ("4096<d<=8192, span<=2^18", (dplus > 4096) & (dplus <= 8192) & (span <= 2**18)),
                  ("4096<d<=8192, span>2^18", (dplus > 4096) & (dplus <= 8192) & (span > 2**18)),
                  ("d>8192", dplus > 8192)]:
    mm = c3 & msk
    print(f"  {name}: heads {int(mm.sum())}, work {float(W[mm].sum()):.3e}, in-edges {int(din[mm].sum())}")
