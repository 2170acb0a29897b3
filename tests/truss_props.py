"""Size-independent properties of a truss decomposition (test helper; no oracle
or libgc code).

For the trussness tau of P:299-302 (tau(e) = the largest k whose k-truss holds
e; every edge of a k-truss lies in >= k-2 of its triangles) write
kappa = tau - 2.  Then for every edge e

    kappa(e) = H({ min(kappa(f), kappa(g)) : (e, f, g) a triangle of G }),

H the h-index (the largest h with >= h values >= h):
  * ">=" side: e lies in the tau(e)-truss, so >= kappa(e) of its triangles
    have both other edges at trussness >= tau(e)           (soundness);
  * "<=" side: were there h = kappa(e)+1 triangles whose other edges are in
    the (h+2)-truss, that truss plus e would be an (h+2)-truss holding e
    (maximality, "maximal").
A value too high or too low on an edge breaks the identity on that edge or on
a neighbour.  (The identity is necessary, not sufficient: lowering a whole
level consistently can keep it - the exact goldens cover that at C3 / C4.)

Global facts checked on the full arrays: tau >= 2; tau = 2 exactly on the
support-0 edges (the 3-truss is {s >= 1}); tau <= s + 2; kmax = max tau.
"""
from __future__ import annotations

import numpy as np


def h_index(vals: np.ndarray) -> int:
    if vals.size == 0:
        return 0
    s = np.sort(vals)[::-1]
    return int(np.count_nonzero(s >= np.arange(1, s.size + 1)))


def common_edge_ids(ptr, col, eid, a: int, b: int):
    """Edge ids (f, g) of every triangle through {a, b}: f = {a, w}, g = {b, w}
    for w in N(a) & N(b) (sorted rows; the shorter row searched in the longer)."""
    ra, rb = slice(ptr[a], ptr[a + 1]), slice(ptr[b], ptr[b + 1])
    na, nb, ea, eb = col[ra], col[rb], eid[ra], eid[rb]
    if na.size > nb.size:
        na, nb, ea, eb = nb, na, eb, ea
    if na.size == 0:
        return ea[:0], eb[:0]
    pos = np.searchsorted(nb, na)
    pos[pos == nb.size] = nb.size - 1
    hit = nb[pos] == na
    return ea[hit], eb[pos[hit]]


def check_global(sup: np.ndarray, tau: np.ndarray, kmax: int) -> None:
    tau = np.asarray(tau)
    assert tau.size == sup.size
    if tau.size == 0:
        return
    assert int(tau.min()) >= 2
    assert int(tau.max()) == kmax
    assert np.array_equal(tau == 2, sup == 0)              # 3-truss = {s >= 1}
    assert bool((tau.astype(np.int64) <= sup.astype(np.int64) + 2).all())


def sample_edges(tau: np.ndarray, n_uniform: int, n_top: int, per_level: int, seed: int) -> np.ndarray:
    """Seeded sample: uniform edges, the highest-trussness edges, and a few
    edges of every populated level (so small deep levels are not missed)."""
    rng = np.random.default_rng(seed)
    m = tau.size
    picks = [rng.integers(0, m, size=min(n_uniform, m))]
    if n_top:
        picks.append(np.argpartition(tau, max(m - n_top, 0))[max(m - n_top, 0):])
    if per_level:
        order = np.argsort(tau, kind="stable")
        st = tau[order]
        starts = np.flatnonzero(np.r_[True, st[1:] != st[:-1]])
        ends = np.r_[starts[1:], m]
        for s, e in zip(starts, ends):
            take = min(per_level, e - s)
            picks.append(order[s + rng.choice(e - s, size=take, replace=False)])
    return np.unique(np.concatenate(picks))


def check_local(ptr, col, eid, cu, cv, tau: np.ndarray, edges: np.ndarray) -> int:
    """The h-index identity on the given edge ids; returns the number checked."""
    for e in edges.tolist():
        f, g = common_edge_ids(ptr, col, eid, int(cu[e]), int(cv[e]))
        vals = np.minimum(tau[f], tau[g]).astype(np.int64) - 2
        h = h_index(vals)
        assert h == int(tau[e]) - 2, (e, int(cu[e]), int(cv[e]), int(tau[e]), h)
    return int(edges.size)
