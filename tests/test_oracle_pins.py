"""Pins for the CPU oracle (CPU only, ``-m "not gpu"``).

The oracle (oracle/oracle.c) is checked against things other than itself:
values the paper prints (Table II, Fig. 1/2 examples, tests/golden/), closed
forms (K_n, cycles, trees, bipartite graphs), brute-force triple enumeration,
dense linear algebra (trace(A^3)/6, A^2 on edges), the paper's own array
algorithms run literally in scipy (Alg. 1-4), networkx, and
invariants.  A dropped term, a wrong bound or a
double-counted triangle in the oracle fails at least one of these.
"""
from __future__ import annotations

import itertools
import json
import math
import os

import networkx as nx
import numpy as np
import pytest
import scipy.sparse as sp
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import gen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------- helpers --
def random_simple_graph(n, p, rng):
    """Edge list (a<b) of G(n,p) from numpy's RNG (independent of gen/)."""
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(iu.size) < p
    return iu[keep].astype(np.int32), ju[keep].astype(np.int32)


def noisy(u, v, rng, n):
    """Raw list with duplicates, reversed copies and self-loops added."""
    k = u.size
    parts_u = [u, v[: k // 2], u[: k // 3]]
    parts_v = [v, u[: k // 2], v[: k // 3]]
    loops = rng.integers(0, max(n, 1), size=3).astype(np.int32)
    parts_u.append(loops)
    parts_v.append(loops)
    U = np.concatenate(parts_u)
    V = np.concatenate(parts_v)
    perm = rng.permutation(U.size)
    return U[perm], V[perm]


def brute_force(n, edges):
    """O(n^3) triple enumeration: triangles and per-edge apex counts."""
    adj = [[False] * n for _ in range(n)]
    for a, b in edges:
        adj[a][b] = adj[b][a] = True
    T = 0
    for a, b, c in itertools.combinations(range(n), 3):
        if adj[a][b] and adj[b][c] and adj[a][c]:
            T += 1
    sup = [sum(1 for w in range(n) if adj[a][w] and adj[b][w]) for a, b in edges]
    return T, sup


def dense_adj(g):
    A = np.zeros((g.n, g.n), dtype=np.int64)
    A[g.cu, g.cv] = 1
    A[g.cv, g.cu] = 1
    return A


def alg4_literal(g, k):
    """PAPER.md Algorithm 4 executed literally on scipy matrices.

    E is the m x n unoriented incidence matrix (rows = edges);
    d = sum(E) is MATLAB's column sum (reading A13).  Returns the surviving
    original edge ids."""
    m, n = g.m, g.n
    rows = np.repeat(np.arange(m), 2)
    cols = np.stack([g.cu, g.cv], axis=1).ravel()
    E = sp.csr_matrix((np.ones(2 * m, dtype=np.int64), (rows, cols)), shape=(m, n))
    ids = np.arange(m)
    d = np.asarray(E.sum(axis=0)).ravel()
    A = (E.T @ E - sp.diags(d, dtype=np.int64)).tocsr()
    R = (E @ A).tocsr()
    s = np.asarray((R == 2).sum(axis=1)).ravel()
    x = np.flatnonzero(s < k - 2)
    while x.size > 0:
        xc = np.setdiff1d(np.arange(E.shape[0]), x)
        Ex = E[x, :]
        E = E[xc, :]
        ids = ids[xc]
        dx = np.asarray(Ex.sum(axis=0)).ravel()
        R = R[xc, :]
        R = (R - E @ (Ex.T @ Ex - sp.diags(dx, dtype=np.int64))).tocsr()
        R.eliminate_zeros()
        s = np.asarray((R == 2).sum(axis=1)).ravel()
        x = np.flatnonzero(s < k - 2)
    return set(ids.tolist())


def alg4_scratch_R(g, alive_ids):
    """R = E A recomputed from scratch on a subset of edges (for A5's identity)."""
    sub = np.array(sorted(alive_ids), dtype=np.int64)
    m2 = sub.size
    rows = np.repeat(np.arange(m2), 2)
    cols = np.stack([g.cu[sub], g.cv[sub]], axis=1).ravel()
    E = sp.csr_matrix((np.ones(2 * m2, dtype=np.int64), (rows, cols)), shape=(m2, g.n))
    d = np.asarray(E.sum(axis=0)).ravel()
    A = (E.T @ E - sp.diags(d, dtype=np.int64)).tocsr()
    return (E @ A).toarray()


def nx_graph(g):
    G = nx.Graph()
    G.add_nodes_from(range(g.n))
    G.add_edges_from(zip(g.cu.tolist(), g.cv.tolist()))
    return G


def edge_index(g):
    return {(int(a), int(b)): i for i, (a, b) in enumerate(zip(g.cu, g.cv))}


# ------------------------------------------------------------------ sorting --
def test_sort_u64_matches_numpy():
    rng = np.random.default_rng(0)
    for n in [0, 1, 2, 7, 1000, 100_000]:
        k = rng.integers(0, 2**63, size=n, dtype=np.uint64)
        k[: n // 3] = k[n // 2: n // 2 + n // 3] if n > 6 else k[: n // 3]   # duplicates
        assert np.array_equal(oracle.sort_u64(k), np.sort(k))
    k = np.full(50, 12345, dtype=np.uint64)
    assert np.array_equal(oracle.sort_u64(k), k)


# ------------------------------------------------------------ O-1 / O-2 ----
def test_canonicalize_matches_set_definition():
    rng = np.random.default_rng(1)
    for trial in range(20):
        n = int(rng.integers(1, 60))
        u = rng.integers(0, n, size=200).astype(np.int32)
        v = rng.integers(0, n, size=200).astype(np.int32)
        g = oracle.OracleGraph(u, v)
        want = sorted({(min(a, b), max(a, b)) for a, b in zip(u.tolist(), v.tolist()) if a != b})
        assert list(zip(g.cu.tolist(), g.cv.tolist())) == want
        assert g.n == int(max(u.max(), v.max())) + 1
        # adjacency rows sorted, symmetric, eids consistent
        for x in range(g.n):
            row = g.col[g.ptr[x]: g.ptr[x + 1]]
            assert np.all(np.diff(row) > 0)
            for w, e in zip(row, g.eid[g.ptr[x]: g.ptr[x + 1]]):
                assert {int(g.cu[e]), int(g.cv[e])} == {x, int(w)}


def test_canonicalize_edge_cases():
    g = oracle.OracleGraph([], [])
    assert (g.n, g.m) == (0, 0)
    assert g.triangle_count() == 0
    g = oracle.OracleGraph([3, 3, 5], [3, 3, 5])          # only self loops
    assert (g.n, g.m) == (6, 0)
    tau, kmax = g.truss_decomposition()
    assert kmax == 0 and tau.size == 0                      # reading A7
    with pytest.raises(ValueError):
        oracle.OracleGraph([0, -1], [1, 2])


def test_normalization_property():
    """P12 / P:134-136: duplicates, reversed copies and self-loops change nothing."""
    rng = np.random.default_rng(2)
    u, v = random_simple_graph(40, 0.2, rng)
    g0 = oracle.OracleGraph(u, v)
    U, V = noisy(u, v, rng, 40)
    g1 = oracle.OracleGraph(U, V)
    assert np.array_equal(g0.cu, g1.cu) and np.array_equal(g0.cv, g1.cv)
    g2 = oracle.OracleGraph(g1.cu, g1.cv)                   # idempotent
    assert np.array_equal(g1.cu, g2.cu) and np.array_equal(g1.cv, g2.cv)


# --------------------------------------------------- paper worked examples --
@pytest.mark.parametrize("fixture", ["fig1_diamond.json", "k4_ear.json", "pendant_triangle.json",
                                     "hub_two_k4.json"])
def test_golden_examples(fixture):
    d = json.load(open(os.path.join(GOLDEN, fixture)))
    g = oracle.OracleGraph(d["raw_u"], d["raw_v"])
    assert g.cu.tolist() == d["canonical_u"] and g.cv.tolist() == d["canonical_v"]
    assert g.triangle_count() == d["triangles"]
    assert g.support().tolist() == d["support"]
    for k, mask in d["ktruss"].items():
        alive, _ = g.ktruss(int(k))
        assert alive.tolist() == mask, (fixture, k)
    tau, kmax = g.truss_decomposition()
    assert tau.tolist() == d["trussness"] and kmax == d["kmax"]
    tau2, kmax2 = g.truss_sequential()
    assert tau2.tolist() == d["trussness"] and kmax2 == d["kmax"]
    tau3, kmax3 = g.truss_parallel()
    assert tau3.tolist() == d["trussness"] and kmax3 == d["kmax"]


def test_k4_ear_needs_single_decrement():
    """Reading A5: edges (0,4),(1,4) leave in one round; triangle (0,1,4) costs (0,1) once."""
    d = json.load(open(os.path.join(GOLDEN, "k4_ear.json")))
    g = oracle.OracleGraph(d["raw_u"], d["raw_v"])
    alive, trace = g.ktruss(4)
    assert trace.tolist() == [2]                            # one batch round removes both
    assert int(alive.sum()) == 6


# ------------------------------------------------------------ closed forms --
@pytest.mark.parametrize("n", [3, 4, 5, 7, 10, 13])
def test_complete_graph_closed_form(n):
    """P2: K_n has C(n,3) triangles, every support n-2, k-truss = K_n iff k <= n."""
    u, v = zip(*itertools.combinations(range(n), 2))
    g = oracle.OracleGraph(list(u), list(v))
    assert g.triangle_count() == math.comb(n, 3)
    assert np.all(g.support() == n - 2)
    for k in range(2, n + 3):
        alive, _ = g.ktruss(k)
        assert alive.all() if k <= n else not alive.any()
    tau, kmax = g.truss_decomposition()
    assert np.all(tau == n) and kmax == n
    tau2, kmax2 = g.truss_sequential()
    assert np.all(tau2 == n) and kmax2 == n
    tau3, kmax3 = g.truss_parallel()
    assert np.all(tau3 == n) and kmax3 == n


def _triangle_free_cases():
    cases = {}
    for n in [4, 5, 9, 64]:                                 # cycles C_n, n >= 4
        cases[f"cycle{n}"] = ([i for i in range(n)], [(i + 1) % n for i in range(n)])
    cases["path50"] = (list(range(49)), list(range(1, 50)))
    cases["star100"] = ([0] * 99, list(range(1, 100)))
    rng = np.random.default_rng(3)
    par = [int(rng.integers(0, i)) for i in range(1, 200)]  # random tree
    cases["tree200"] = (par, list(range(1, 200)))
    a, b = 5, 7                                             # complete bipartite K_{5,7}
    cases["K5_7"] = ([i for i in range(a) for _ in range(b)], [a + j for _ in range(a) for j in range(b)])
    return cases


@pytest.mark.parametrize("name", sorted(_triangle_free_cases()))
def test_triangle_free_closed_form(name):
    """P3: cycles (n>=4), paths, stars, trees, bipartite graphs: T = 0, S = 0,
    3-truss empty, every trussness 2, kmax = 2."""
    u, v = _triangle_free_cases()[name]
    g = oracle.OracleGraph(u, v)
    assert g.m > 0
    assert g.triangle_count() == 0
    assert not g.support().any()
    alive, _ = g.ktruss(3)
    assert not alive.any()
    alive, _ = g.ktruss(2)
    assert alive.all()                                      # k = 2: vacuous (A3)
    tau, kmax = g.truss_decomposition()
    assert np.all(tau == 2) and kmax == 2


def test_ktruss_rejects_k_below_2():
    g = oracle.OracleGraph([0, 1, 2], [1, 2, 0])
    with pytest.raises(ValueError):
        g.ktruss(1)


# ------------------------------------------------------------ Table II -----
def _table2():
    rows = []
    for line in open(os.path.join(GOLDEN, "table2_king_grid.tsv")):
        if line.startswith("#") or not line.strip():
            continue
        rows.append(tuple(int(x) for x in line.split()))
    return rows


def test_king_grid_small_bruteforce():
    """P10: every triangle of the king graph lies in one 2x2 cell: 4(M-1)^2."""
    for M in range(2, 9):
        u, v = gen.king_grid(M)
        g = oracle.OracleGraph(u, v)
        edges = list(zip(g.cu.tolist(), g.cv.tolist()))
        T, sup = brute_force(g.n, edges)
        assert g.m == 2 * (M - 1) * (2 * M - 1)
        assert g.triangle_count() == T == 4 * (M - 1) ** 2
        assert g.support().tolist() == sup


@pytest.mark.parametrize("row", _table2()[:2])
def test_king_grid_table2(row):
    """Table II: node and edge counts exact; the triangle column is
    2x the 3-clique count (reading A9)."""
    nexp, nodes, edges, tri_printed = row
    M = 2 ** nexp
    u, v = gen.king_grid(M)
    g = oracle.OracleGraph(u, v)
    assert g.n == nodes == M * M
    assert g.m == edges
    T = g.triangle_count()
    assert 2 * T == tri_printed
    assert int(g.support().sum()) == 3 * T


def test_table2_closed_forms_all_rows():
    for nexp, nodes, edges, tri in _table2():
        M = 2 ** nexp
        assert nodes == M * M and edges == 2 * (M - 1) * (2 * M - 1) and tri == 8 * (M - 1) ** 2


# --------------------------------------------------- brute force / dense --
def test_bruteforce_random_graphs():
    rng = np.random.default_rng(4)
    for trial in range(25):
        n = int(rng.integers(3, 30))
        u, v = random_simple_graph(n, float(rng.uniform(0.1, 0.9)), rng)
        U, V = noisy(u, v, rng, n)
        g = oracle.OracleGraph(U, V)
        edges = list(zip(g.cu.tolist(), g.cv.tolist()))
        T, sup = brute_force(max(g.n, 1), edges)
        assert g.triangle_count() == T
        assert g.support().tolist() == sup


def test_c1_full_bruteforce_and_trace():
    """C1 in full: per-edge apex counts by dense bitset rows, T = trace(A^3)/6,
    support(u,v) = (A^2)(u,v) on edges (P5; Alg. 2's C = A^2 ∘ A)."""
    u, v = gen.CONFIGS["C1"].generate()
    g = oracle.OracleGraph(u, v)
    A = dense_adj(g)
    B = A.astype(bool)
    sup_bits = np.array([int(np.count_nonzero(B[a] & B[b])) for a, b in zip(g.cu, g.cv)])
    A2 = A @ A
    T = int(np.trace(A2 @ A)) // 6
    assert g.triangle_count() == T
    assert np.array_equal(g.support(), sup_bits)
    assert np.array_equal(g.support(), A2[g.cu, g.cv])


def test_dense_trace_random():
    rng = np.random.default_rng(5)
    for n in [50, 200, 400]:
        u, v = random_simple_graph(n, 0.1, rng)
        g = oracle.OracleGraph(u, v)
        A = dense_adj(g)
        assert g.triangle_count() == int(np.trace(A @ A @ A)) // 6


# -------------------------------------------- the paper's array algorithms --
def _some_graphs():
    rng = np.random.default_rng(6)
    out = []
    for trial in range(12):
        n = int(rng.integers(6, 40))
        u, v = random_simple_graph(n, float(rng.uniform(0.15, 0.6)), rng)
        out.append(oracle.OracleGraph(u, v))
    out.append(oracle.OracleGraph(*gen.rmat(7, 8, seed=11)))
    return out


def test_alg1_alg2_alg3_literal():
    """Alg. 1 (C = AE overloaded; nnz(C)/3, column counts = support), Alg. 2
    (sum(A^2 ∘ A)/6), Alg. 3 (sum(A ∘ LU)/2)."""
    for g in _some_graphs():
        A = sp.csr_matrix(dense_adj(g))
        m = g.m
        # Alg. 1 with E as n x m (P:196 indexes E(x,j), reading A12):
        E = sp.csr_matrix((np.ones(2 * m, dtype=np.int64),
                           (np.concatenate([g.cu, g.cv]), np.concatenate([np.arange(m), np.arange(m)]))),
                          shape=(g.n, m))
        AE = (A @ E).toarray()                   # AE(i,j) = A(i,x) + A(i,y) for edge j = (x,y)
        C1 = AE == 2                             # C(i,j) = {i,x,y} iff both adjacent
        assert int(C1.sum()) // 3 == g.triangle_count()
        assert np.array_equal(C1.sum(axis=0), g.support())
        # Alg. 2
        C2 = (A @ A).multiply(A)
        assert int(C2.sum()) // 6 == g.triangle_count()
        assert np.array_equal(np.asarray(C2[g.cu, g.cv]).ravel(), g.support())
        # Alg. 3
        L = sp.tril(A, -1).tocsr()
        U = sp.triu(A, 1).tocsr()
        C3 = A.multiply(L @ U)
        assert int(C3.sum()) // 2 == g.triangle_count()


def test_alg4_literal_matches_ktruss():
    """Alg. 4 run literally == oracle O-5 for k = 2..8."""
    for g in _some_graphs():
        for k in range(2, 9):
            want = alg4_literal(g, k)
            alive, _ = g.ktruss(k)
            assert set(np.flatnonzero(alive).tolist()) == want, (g.n, g.m, k)


def test_alg4_recompute_identity():
    """A = E^T E - diag(E^T E) lets R = EA be updated after a removal
    instead of recomputed; the updated R equals the scratch R."""
    rng = np.random.default_rng(7)
    u, v = random_simple_graph(25, 0.35, rng)
    g = oracle.OracleGraph(u, v)
    m = g.m
    rows = np.repeat(np.arange(m), 2)
    cols = np.stack([g.cu, g.cv], axis=1).ravel()
    E = sp.csr_matrix((np.ones(2 * m, dtype=np.int64), (rows, cols)), shape=(m, g.n))
    d = np.asarray(E.sum(axis=0)).ravel()
    A = E.T @ E - sp.diags(d, dtype=np.int64)
    R = (E @ A).tocsr()
    x = rng.choice(m, size=m // 4, replace=False)
    xc = np.setdiff1d(np.arange(m), x)
    Ex, Ek = E[x, :], E[xc, :]
    dx = np.asarray(Ex.sum(axis=0)).ravel()
    R2 = (R[xc, :] - Ek @ (Ex.T @ Ex - sp.diags(dx, dtype=np.int64))).toarray()
    assert np.array_equal(R2, alg4_scratch_R(g, xc.tolist()))


# ---------------------------------------------------------------- networkx --
def test_networkx_triangles_and_ktruss():
    graphs = _some_graphs() + [oracle.OracleGraph(*gen.CONFIGS["C1"].generate())]
    for g in graphs:
        G = nx_graph(g)
        assert sum(nx.triangles(G).values()) // 3 == g.triangle_count()
        idx = edge_index(g)
        for k in [3, 4, 5, 6]:
            H = nx.k_truss(G, k)
            want = {idx[(min(a, b), max(a, b))] for a, b in H.edges()}
            alive, _ = g.ktruss(k)
            assert set(np.flatnonzero(alive).tolist()) == want, (g.n, k)


# -------------------------------------------------------------- invariants --
def test_permutation_invariance():
    rng = np.random.default_rng(8)
    u, v = gen.rmat(9, 8, seed=21)
    g = oracle.OracleGraph(u, v)
    perm = rng.permutation(g.n).astype(np.int32)
    h = oracle.OracleGraph(perm[u], perm[v])
    assert h.triangle_count() == g.triangle_count()
    hidx = edge_index(h)
    sup_h = h.support()
    mapped = np.array([sup_h[hidx[(min(perm[a], perm[b]), max(perm[a], perm[b]))]] for a, b in zip(g.cu, g.cv)])
    assert np.array_equal(mapped, g.support())
    tg, kg = g.truss_decomposition()
    th, kh = h.truss_decomposition()
    assert kg == kh
    mapped_t = np.array([th[hidx[(min(perm[a], perm[b]), max(perm[a], perm[b]))]] for a, b in zip(g.cu, g.cv)])
    assert np.array_equal(mapped_t, tg)


def test_edge_deletion_drops_support():
    """T(G) - T(G - e) = support(e)."""
    rng = np.random.default_rng(9)
    u, v = random_simple_graph(35, 0.3, rng)
    g = oracle.OracleGraph(u, v)
    T = g.triangle_count()
    sup = g.support()
    for e in rng.choice(g.m, size=10, replace=False):
        keep = np.arange(g.m) != e
        h = oracle.OracleGraph(g.cu[keep], g.cv[keep])
        assert T - h.triangle_count() == sup[e]


def test_truss_properties_and_tiers_agree():
    """Nesting, fixed point, in-truss support >= k-2, O-6 == O-7,
    decomposition consistent with every ktruss(k)."""
    graphs = _some_graphs() + [oracle.OracleGraph(*gen.CONFIGS["C1"].generate())]
    for g in graphs:
        tau, kmax = g.truss_decomposition()
        tau2, kmax2 = g.truss_sequential()
        assert np.array_equal(tau, tau2) and kmax == kmax2
        tau3, kmax3 = g.truss_parallel()
        assert np.array_equal(tau, tau3) and kmax == kmax3
        prev = None
        for k in range(2, kmax + 2):
            alive, _ = g.ktruss(k)
            assert np.array_equal(alive.astype(bool), tau >= k)
            if prev is not None:
                assert not np.any(alive & ~prev)                       # nesting
            sub = np.flatnonzero(alive)
            if sub.size:
                h = oracle.OracleGraph(g.cu[sub], g.cv[sub])
                assert np.all(h.support() >= k - 2)                    # truss condition
                again, _ = h.ktruss(k)
                assert again.all()                                      # fixed point
            prev = alive
        assert not g.ktruss(kmax + 1)[0].any()


def test_c1_truss_decomposition_against_networkx():
    g = oracle.OracleGraph(*gen.CONFIGS["C1"].generate())
    tau, kmax = g.truss_decomposition()
    G = nx_graph(g)
    idx = edge_index(g)
    H = nx.k_truss(G, kmax)
    assert H.number_of_edges() > 0 and nx.k_truss(G, kmax + 1).number_of_edges() == 0
    assert {idx[(min(a, b), max(a, b))] for a, b in H.edges()} == set(np.flatnonzero(tau == kmax).tolist())


def test_thread_count_independence():
    u, v = gen.rmat(12, 16, seed=31)
    g1 = oracle.OracleGraph(u, v, nthreads=1)
    g8 = oracle.OracleGraph(u, v, nthreads=8)
    assert np.array_equal(g1.support(), g8.support())
    assert g1.triangle_count() == g8.triangle_count()


def test_c2_statistics():
    """P13: statistical sanity only (E[m] = p C(n,2), E[T] = C(n,3) p^3), not parity."""
    g = oracle.OracleGraph(*gen.CONFIGS["C2"].generate())
    n = 65536
    p = 32.0 / (n - 1)
    em = p * n * (n - 1) / 2
    assert abs(g.m - em) < 6 * math.sqrt(em)
    et = math.comb(n, 3) * p ** 3
    assert 0.8 * et < g.triangle_count() < 1.2 * et


# -------------------------------------------------------------- hypothesis --
@st.composite
def raw_graphs(draw):
    n = draw(st.integers(1, 24))
    k = draw(st.integers(0, 120))
    u = draw(st.lists(st.integers(0, n - 1), min_size=k, max_size=k))
    v = draw(st.lists(st.integers(0, n - 1), min_size=k, max_size=k))
    return np.array(u, dtype=np.int32), np.array(v, dtype=np.int32)


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(raw_graphs())
def test_hypothesis_oracle(raw):
    u, v = raw
    g = oracle.OracleGraph(u, v)
    edges = list(zip(g.cu.tolist(), g.cv.tolist()))
    T, sup = brute_force(max(g.n, 1), edges)
    assert g.triangle_count() == T
    assert g.support().tolist() == sup
    tau, kmax = g.truss_decomposition()
    tau2, kmax2 = g.truss_sequential()
    assert np.array_equal(tau, tau2) and kmax == kmax2
    tau3, kmax3 = g.truss_parallel()
    assert np.array_equal(tau, tau3) and kmax == kmax3
    tau3, kmax3 = g.truss_parallel()
    assert np.array_equal(tau, tau3) and kmax == kmax3
    if g.m:
        G = nx_graph(g)
        idx = edge_index(g)
        for k in (3, 4):
            want = {idx[(min(a, b), max(a, b))] for a, b in nx.k_truss(G, k).edges()}
            assert set(np.flatnonzero(tau >= k).tolist()) == want


# ------------------------------------------------------- file formats --
def test_tsv_and_mmio_round_trip(tmp_path):
    """Graph Challenge TSV triples and MMIO coordinate files, 1-based on disk,
    0-based pairs in memory; the oracle sees the same graph either way."""
    from paper_1708_06866_b200 import io as gio
    u, v = gen.rmat(9, 8, seed=11)
    p = str(tmp_path / "g.tsv")
    gio.write_tsv(p, u, v)
    first = open(p).readline().split("\t")
    assert int(first[0]) == u[0] + 1 and int(first[1]) == v[0] + 1 and first[2].strip() == "1"
    ru, rv = gio.read_tsv(p)
    assert np.array_equal(ru, u) and np.array_equal(rv, v)
    q = str(tmp_path / "g.mtx")
    gio.write_mmio(q, u, v)
    mu, mv = gio.read_mmio(q)
    assert np.array_equal(mu, u) and np.array_equal(mv, v)
    assert oracle.OracleGraph(ru, rv).triangle_count() == oracle.OracleGraph(u, v).triangle_count()
    with open(str(tmp_path / "bad.tsv"), "w") as f:
        f.write("0\t3\t1\n")
    with pytest.raises(ValueError):
        gio.read_tsv(str(tmp_path / "bad.tsv"))


def test_king_grid_configs_match_table2():
    """K12 / K13 bench workloads are Table II rows 12 and 13."""
    rows = {}
    for line in open(os.path.join(GOLDEN, "table2_king_grid.tsv")):
        if line.startswith("#") or not line.strip():
            continue
        nn, nodes, edges, tri = (int(x) for x in line.split())
        rows[nn] = (nodes, edges, tri)
    for name, nn in (("K12", 12), ("K13", 13)):
        cfg = gen.CONFIGS[name]
        assert cfg.n == 2 ** nn and cfg.n ** 2 == rows[nn][0]
        assert 2 * (cfg.n - 1) * (2 * cfg.n - 1) == rows[nn][1]


# ------------------------------------------- skewed pairs (galloping branches) --
@st.composite
def hub_graphs(draw):
    """A random core (n <= 16) plus a hub whose degree is >= 32x every core
    degree: the hub joins a random subset of the core and enough outside
    vertices, some of which are joined to each other and to the core, so
    hub-core pairs take the oracle's binary-search branches (O-3, O-5, O-7)
    while the hub's triangles die and live in every combination."""
    n = draw(st.integers(3, 16))
    pairs = [(a, b) for a in range(n) for b in range(a + 1, n)]
    core = draw(st.lists(st.sampled_from(pairs), max_size=len(pairs), unique=True))
    hub = n
    joins = draw(st.lists(st.integers(0, n - 1), min_size=1, max_size=n, unique=True))
    npend = 32 * n + draw(st.integers(0, 40))
    first = n + 1
    extra = draw(st.lists(st.tuples(st.integers(0, npend - 1), st.integers(0, npend - 1)), max_size=12))
    cross = draw(st.lists(st.tuples(st.integers(0, npend - 1), st.integers(0, n - 1)), max_size=6))
    u = [a for a, _ in core] + [hub] * len(joins) + [hub] * npend
    v = [b for _, b in core] + joins + list(range(first, first + npend))
    u += [first + a for a, _ in extra] + [first + a for a, _ in cross]
    v += [first + b for _, b in extra] + [b for _, b in cross]
    return np.array(u, np.int32), np.array(v, np.int32)


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(hub_graphs())
def test_hypothesis_hub_graphs(raw):
    """Degree ratios >= 32: supports = (A^2)(u,v), T =
    trace(A^3)/6, k-trusses = networkx for k = 3..5, O-6 == O-7."""
    u, v = raw
    g = oracle.OracleGraph(u, v)
    A = dense_adj(g)
    A2 = A @ A
    assert g.triangle_count() == int(np.trace(A2 @ A)) // 6
    assert np.array_equal(g.support(), A2[g.cu, g.cv])
    G = nx_graph(g)
    idx = edge_index(g)
    for k in (3, 4, 5):
        want = {idx[(min(a, b), max(a, b))] for a, b in nx.k_truss(G, k).edges()}
        alive, _ = g.ktruss(k)
        assert set(np.flatnonzero(alive).tolist()) == want, k
    tau, kmax = g.truss_decomposition()
    tau2, kmax2 = g.truss_sequential()
    assert np.array_equal(tau, tau2) and kmax == kmax2
    tau3, kmax3 = g.truss_parallel()
    assert np.array_equal(tau, tau3) and kmax == kmax3


# ------------------------------------------ k-truss byte-model terms (§8(d)) --
def _batch_replay_work(edges, k):
    """Plain-Python replay of Alg. 4's batch rounds on an edge set:
    sum over rounds of min(d(a), d(b)) for x-edges with support > 0 (alive
    degrees at the round start) and D = the support lost by edges that stay."""
    alive = set(edges)
    sum_min = dec = 0
    prev = None
    while True:
        nb = {}
        for a, b in alive:
            nb.setdefault(a, set()).add(b)
            nb.setdefault(b, set()).add(a)
        s = {e: len(nb[e[0]] & nb[e[1]]) for e in alive}
        if prev is not None:
            dec += sum(prev[e] - s[e] for e in alive)
        x = {e for e in alive if s[e] < k - 2}
        if not x:
            return sum_min, dec
        sum_min += sum(min(len(nb[a]), len(nb[b])) for a, b in x if s[(a, b)] > 0)
        prev = s
        alive -= x


def test_ktruss_work_terms_fixtures():
    """Hand-derived (DESIGN.md §7 "k-truss roofline"): K4+ear at k = 4: round 1
    removes (0,4), (1,4), min degrees 2 + 2, triangle (0,1,4) costs (0,1) one
    unit; the hub fixture at k = 4: (w1,H), (w2,H) with min degree 4 each, the
    two hub triangles cost 2 units each; the decompositions add every later
    level's rounds; K_n at k = n+1: every edge in round 1, min degree n-1, no
    survivor to decrement."""
    d = json.load(open(os.path.join(GOLDEN, "k4_ear.json")))
    g = oracle.OracleGraph(d["raw_u"], d["raw_v"])
    assert g.ktruss(4, work=True)[2] == {"sum_min": 4, "decrements": 1}
    assert g.truss_decomposition(work=True)[2] == {"sum_min": 4 + 6 * 3, "decrements": 1}
    d = json.load(open(os.path.join(GOLDEN, "hub_two_k4.json")))
    g = oracle.OracleGraph(d["raw_u"], d["raw_v"])
    assert g.ktruss(4, work=True)[2] == {"sum_min": 8, "decrements": 4}
    assert g.truss_decomposition(work=True)[2] == {"sum_min": 3 + 3 + 12 * 3, "decrements": 4}
    for n in (4, 7, 12):
        u, v = zip(*itertools.combinations(range(n), 2))
        g = oracle.OracleGraph(list(u), list(v))
        assert g.ktruss(n + 1, work=True)[2] == {"sum_min": math.comb(n, 2) * (n - 1), "decrements": 0}
        assert g.ktruss(n, work=True)[2] == {"sum_min": 0, "decrements": 0}


def test_ktruss_work_terms_bruteforce():
    rng = np.random.default_rng(12)
    graphs = [oracle.OracleGraph(*random_simple_graph(int(rng.integers(5, 40)), float(rng.uniform(0.1, 0.6)), rng))
              for _ in range(15)]
    graphs.append(oracle.OracleGraph(*gen.rmat(7, 8, seed=12)))
    for g in graphs:
        edges = list(zip(g.cu.tolist(), g.cv.tolist()))
        tot = [0, 0]
        for k in range(3, 9):
            w = g.ktruss(k, work=True)[2]
            assert (w["sum_min"], w["decrements"]) == _batch_replay_work(edges, k), k
        # decomposition: k = 3, 4, ... each from the previous survivors
        tau, kmax, wd = g.truss_decomposition(work=True)
        for k in range(3, kmax + 2):
            surv = [e for e, t in zip(edges, tau.tolist()) if t >= k - 1]
            sm, dc = _batch_replay_work(surv, k)
            tot[0] += sm
            tot[1] += dc
        assert (wd["sum_min"], wd["decrements"]) == tuple(tot)


def test_tier2_decompositions_larger_graphs():
    """O-7 (sequential bucket peel) and O-8 (parallel incremental rounds) equal
    O-6 (batch recompute, the definition) on R-MAT graphs with deep cores and a
    skewed one, and O-8 does not depend on the thread count."""
    for s, ef, seed, abc in [(12, 16, 5, (0.57, 0.19, 0.19)), (13, 8, 6, (0.65, 0.15, 0.15)),
                             (11, 32, 7, (0.57, 0.19, 0.19))]:
        u, v = gen.rmat(s, ef, *abc, seed=seed)
        g = oracle.OracleGraph(u, v)
        tau, kmax = g.truss_decomposition()
        assert (g.truss_sequential()[0] == tau).all()
        t8, k8 = g.truss_parallel()
        assert np.array_equal(t8, tau) and k8 == kmax
        g1 = oracle.OracleGraph(u, v, nthreads=1)
        assert np.array_equal(g1.truss_parallel()[0], tau)


def test_o8_checkpoint_resume(tmp_path):
    """O-8 saved at every level start and resumed, call after call (the
    run-time bookkeeping make_golden.py uses for C5), equals O-8 in one call
    and O-6, the definition: the resumed live list and rows (rebuilt from the
    saved edge states) change no result."""
    u, v = gen.rmat(12, 16, 0.57, 0.19, 0.19, seed=5)
    g = oracle.OracleGraph(u, v)
    tau, kmax = g.truss_decomposition()
    sup = g.support()
    ck = str(tmp_path / "o8.ckpt")
    calls, res = 0, None
    while res is None:
        gg = oracle.OracleGraph(u, v)                # a fresh process would rebuild the graph
        res = gg.truss_parallel(sup, consume=True, ckpt=ck, budget_s=1e-9)
        calls += 1
        if res is None:
            # the saved state is an exact partial answer (what make_golden.py stores when O-8 stops at
            # its deadline): removed edges hold their final trussness, live ones have trussness >= k - 1
            k_next = int(np.fromfile(ck, dtype=np.int64, count=7)[3])
            st = np.fromfile(ck, dtype=np.uint8, count=g.m, offset=56 + 4 * g.m)
            tp = np.fromfile(ck, dtype=np.int32, count=g.m, offset=56 + 5 * g.m)
            assert np.array_equal(np.where(st == 0, tp, k_next - 1), np.minimum(tau, k_next - 1))
    assert calls > 3                                  # it really stopped and resumed
    assert np.array_equal(res[0], tau) and res[1] == kmax
    one = oracle.OracleGraph(u, v).truss_parallel(sup)
    assert np.array_equal(one[0], tau) and one[1] == kmax


def test_trussness_h_index_identity():
    """Pin of O-6 / O-7 / O-8 from the definitions alone:
    kappa = tau - 2 is a fixed point of kappa(e) = H({min(kappa(f), kappa(g))})
    over the triangles (e, f, g), H the h-index (tests/truss_props.py: soundness
    one way, maximality the other) - checked on every edge of C1, a skewed
    R-MAT and a hub graph; and the checker rejects a trussness raised or
    lowered on one edge (it is what test_c5_full applies to the GPU's tau)."""
    import truss_props as tp
    hub_u = np.r_[np.zeros(400, np.int32), np.arange(1, 40, dtype=np.int32)]
    hub_v = np.r_[np.arange(1, 401, dtype=np.int32), np.arange(2, 41, dtype=np.int32)]
    graphs = [gen.CONFIGS["C1"].generate(), gen.rmat(11, 16, 0.65, 0.15, 0.15, seed=8), (hub_u, hub_v)]
    for u, v in graphs:
        g = oracle.OracleGraph(u, v)
        sup = g.support()
        for tau, kmax in (g.truss_decomposition(), g.truss_parallel(), g.truss_sequential()):
            tp.check_global(sup, tau, kmax)
            assert tp.check_local(g.ptr, g.col, g.eid, g.cu, g.cv, tau, np.arange(g.m)) == g.m
    # the checker's own teeth, on the last graphs' trussness
    u, v = graphs[0]
    g = oracle.OracleGraph(u, v)
    sup = g.support()
    tau, kmax = g.truss_decomposition()
    rng = np.random.default_rng(4)
    for delta in (+1, -1):
        caught = 0
        cand = np.flatnonzero(tau > 3)
        for e in rng.choice(cand, size=40, replace=False):
            bad = tau.copy()
            bad[e] += delta
            try:
                tp.check_local(g.ptr, g.col, g.eid, g.cu, g.cv, bad, np.array([e]))
            except AssertionError:
                caught += 1
        assert caught == 40, (delta, caught)
    # sampling covers every populated level
    s = tp.sample_edges(tau, 100, 10, 2, seed=1)
    assert set(np.unique(tau[s])) == set(np.unique(tau))
    bad = tau.copy()
    bad[np.flatnonzero(sup == 0)[0]] = 3
    with pytest.raises(AssertionError):
        tp.check_global(sup, bad, kmax)
