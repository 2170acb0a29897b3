"""GPU parity: libgc (through its C ABI) vs the CPU oracle, element by element.

Integer work, so the bar is bit-exact: triangle counts, per-edge supports,
k-truss masks and trussness must equal the oracle's on the same seeded
inputs.  Sizes span several task tiles and ragged tails; every kernel class
is forced over whole graphs; loopback partitions check the multi-GPU split.
"""
from __future__ import annotations

import hashlib
import itertools
import json
import math
import os

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gcmod(gc_lib_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    from paper_1708_06866_b200 import gc
    return gc


@pytest.fixture(scope="module")
def ctx(gcmod):
    c = gcmod.Context(0)
    yield c
    c.close()


def run_gpu(ctx, u, v):
    ctx.load_edges(u, v)
    ctx.build_csr()
    return ctx


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_graph(n, p, rng):
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(iu.size) < p
    u, v = iu[keep].astype(np.int32), ju[keep].astype(np.int32)
    flip = rng.random(u.size) < 0.5
    return np.where(flip, v, u), np.where(flip, u, v)


def check_all(ctx, u, v, ks=(3, 4, 5), decomposition=True):
    g = oracle.OracleGraph(u, v)
    run_gpu(ctx, u, v)
    assert ctx.num_vertices() == g.n
    assert ctx.num_edges() == g.m
    cu, cv = ctx.get_edges()
    assert np.array_equal(cu, g.cu) and np.array_equal(cv, g.cv)
    T = g.triangle_count()
    assert ctx.triangle_count() == T
    sup = ctx.edge_support()
    assert np.array_equal(sup, g.support())
    for k in ks:
        mask, m_alive = ctx.ktruss(k)
        want, _ = g.ktruss(k)
        assert np.array_equal(mask, want), k
        assert m_alive == int(want.sum())
    if decomposition:
        tau, kmax = ctx.truss_decomposition()
        want_tau, want_kmax = g.truss_decomposition()
        assert np.array_equal(tau, want_tau)
        assert kmax == want_kmax
    return g


# ------------------------------------------------------------ paper examples --
@pytest.mark.parametrize("fixture", ["fig1_diamond.json", "k4_ear.json", "pendant_triangle.json",
                                     "hub_two_k4.json"])
def test_golden_examples(ctx, fixture):
    d = json.load(open(os.path.join(GOLDEN, fixture)))
    run_gpu(ctx, np.array(d["raw_u"], np.int32), np.array(d["raw_v"], np.int32))
    cu, cv = ctx.get_edges()
    assert cu.tolist() == d["canonical_u"] and cv.tolist() == d["canonical_v"]
    assert ctx.triangle_count() == d["triangles"]
    assert ctx.edge_support().tolist() == d["support"]
    for k, mask in d["ktruss"].items():
        assert ctx.ktruss(int(k))[0].tolist() == mask
    tau, kmax = ctx.truss_decomposition()
    assert tau.tolist() == d["trussness"] and kmax == d["kmax"]


# ---------------------------------------------------------- degenerate cases --
def test_empty_input(ctx):
    run_gpu(ctx, np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert ctx.num_vertices() == 0 and ctx.num_edges() == 0
    assert ctx.triangle_count() == 0
    assert ctx.edge_support().size == 0
    mask, ma = ctx.ktruss(3)
    assert mask.size == 0 and ma == 0
    tau, kmax = ctx.truss_decomposition()
    assert tau.size == 0 and kmax == 0


def test_only_self_loops(ctx):
    run_gpu(ctx, np.array([4, 4, 1], np.int32), np.array([4, 4, 1], np.int32))
    assert ctx.num_vertices() == 5 and ctx.num_edges() == 0
    assert ctx.triangle_count() == 0
    assert ctx.truss_decomposition()[1] == 0


def test_single_edge_and_duplicates(ctx):
    run_gpu(ctx, np.array([7, 3, 7, 3], np.int32), np.array([3, 7, 3, 3], np.int32))
    assert ctx.num_edges() == 1
    assert ctx.get_edges()[0].tolist() == [3] and ctx.get_edges()[1].tolist() == [7]
    assert ctx.edge_support().tolist() == [0]
    tau, kmax = ctx.truss_decomposition()
    assert tau.tolist() == [2] and kmax == 2


@pytest.mark.parametrize("n", [3, 4, 9, 33, 40, 257, 600])
def test_complete_graphs(ctx, n):
    """K_n closed form (P2): T = C(n,3), S = n-2, tau = n; n spans task classes."""
    u, v = map(np.array, zip(*itertools.combinations(range(n), 2)))
    run_gpu(ctx, u.astype(np.int32), v.astype(np.int32))
    assert ctx.triangle_count() == math.comb(n, 3)
    assert np.all(ctx.edge_support() == n - 2)
    assert ctx.ktruss(n)[1] == n * (n - 1) // 2
    assert ctx.ktruss(n + 1)[1] == 0
    if n <= 257:
        tau, kmax = ctx.truss_decomposition()
        assert np.all(tau == n) and kmax == n


def test_star_cycle_tree(ctx):
    rng = np.random.default_rng(3)
    cases = [([0] * 5000, list(range(1, 5001))),
             (list(range(1000)), [(i + 1) % 1000 for i in range(1000)]),
             ([int(rng.integers(0, i)) for i in range(1, 3000)], list(range(1, 3000)))]
    for u, v in cases:
        run_gpu(ctx, np.array(u, np.int32), np.array(v, np.int32))
        assert ctx.triangle_count() == 0
        assert not ctx.edge_support().any()
        tau, kmax = ctx.truss_decomposition()
        assert np.all(tau == 2) and kmax == 2


# ----------------------------------------------------------- random graphs --
def test_random_small_graphs(ctx):
    rng = np.random.default_rng(11)
    for trial in range(30):
        n = int(rng.integers(2, 70))
        u, v = random_graph(n, float(rng.uniform(0.05, 0.9)), rng)
        extra = rng.integers(0, n, size=(2, 5)).astype(np.int32)   # duplicates / loops
        u = np.concatenate([u, extra[0], extra[0]])
        v = np.concatenate([v, extra[1], extra[0]])
        check_all(ctx, u, v, ks=(2, 3, 4, 5, 6))


def test_fuzz_mixed_structures_and_options(gcmod):
    """Seeded fuzz: planted cliques on a sparse random background with hubs,
    duplicates, reversed pairs, self loops and isolated high ids; every
    result (count, supports, k-truss at random k, decomposition, fused call,
    listing count) against the oracle, under randomly drawn kernel options
    (forced class, task chunk, bitmap, huge-hash limit, long-segment
    threshold, compaction, partitioned peeler, grouped dense-core rounds,
    loopback partitions)."""
    rng = np.random.default_rng(2026)
    for trial in range(40):
        n = int(rng.integers(20, 400))
        u, v = random_graph(n, float(rng.uniform(0.01, 0.08)), rng)
        parts_u, parts_v = [u], [v]
        for _ in range(int(rng.integers(1, 4))):              # planted cliques (deep trusses)
            q = rng.choice(n, size=int(rng.integers(4, min(n, 40))), replace=False).astype(np.int32)
            a, b = np.triu_indices(q.size, 1)
            parts_u.append(q[a]); parts_v.append(q[b])
        hub = int(rng.integers(0, n))                          # a hub joined to a third of the vertices
        nb = rng.choice(n, size=n // 3, replace=False).astype(np.int32)
        parts_u.append(np.full(nb.size, hub, np.int32)); parts_v.append(nb)
        u = np.concatenate(parts_u); v = np.concatenate(parts_v)
        dup = rng.choice(u.size, size=u.size // 5)             # duplicates, both orientations, loops
        u = np.concatenate([u, v[dup], u[:7], np.array([n + 5], np.int32)])
        v = np.concatenate([v, u[dup], u[:7], np.array([n + 9], np.int32)])   # isolated edge far out
        g = oracle.OracleGraph(u, v)
        with gcmod.Context(0) as c:
            loop = int(rng.choice([0, 0, 2, 3]))
            if loop:
                c.comm_init_loopback(loop)
            opts = {gcmod.GC_OPT_TASK_CHUNK: int(rng.choice([64, 777, 32768])),
                    gcmod.GC_OPT_LONG_SEG: int(rng.choice([8, 48, 1 << 30])),
                    gcmod.GC_OPT_BLOCK_BITMAP: int(rng.integers(0, 2)),
                    gcmod.GC_OPT_HUGE_MAX: int(rng.choice([0, 16, 8192])),
                    gcmod.GC_OPT_COMPACT: int(rng.choice([0, 2, 3, 5, 8])),
                    gcmod.GC_OPT_PEEL_PART: int(rng.integers(0, 2)),
                    gcmod.GC_OPT_GROUP_PEEL: int(rng.choice([0, 1, 64, 1 << 20])),
                    gcmod.GC_OPT_GROUP_HEAVY: int(rng.choice([1, 4, 1024])),
                    gcmod.GC_OPT_FORCE_CLASS: int(rng.choice([-1, -1, 1, 2, 3]))}
            c.load_edges(u, v)
            for o, val in opts.items():
                c.set_option(o, val)
            c.build_csr()
            assert c.triangle_count() == g.triangle_count(), (trial, opts)
            assert np.array_equal(c.edge_support(), g.support()), (trial, opts)
            k = int(rng.integers(3, 12))
            want, _ = g.ktruss(k)
            assert np.array_equal(c.ktruss(k)[0], want), (trial, k, opts)
            T, sup, mask, ma = c.ktruss_analysis(k)
            assert T == g.triangle_count() and np.array_equal(sup, g.support()) and np.array_equal(mask, want)
            tau, kmax = c.truss_decomposition()
            want_tau, want_kmax = g.truss_decomposition()
            assert np.array_equal(tau, want_tau) and kmax == want_kmax, (trial, opts)
            assert len(c.list_triangles()) == g.triangle_count()


def test_rmat_small_full(ctx):
    for s, ef, seed in [(8, 8, 5), (11, 16, 6), (12, 4, 7)]:
        u, v = gen.rmat(s, ef, seed=seed)
        check_all(ctx, u, v, ks=(3, 4, 6, 9))


def test_king_grid(ctx):
    """Table II graphs: T = 4(M-1)^2 = Table II / 2 (reading A9)."""
    for M in (5, 64, 256):
        u, v = gen.king_grid(M)
        run_gpu(ctx, u, v)
        assert ctx.num_edges() == 2 * (M - 1) * (2 * M - 1)
        assert ctx.triangle_count() == 4 * (M - 1) ** 2


@pytest.mark.parametrize("name", ["K12", "K13"])
def test_king_grid_table2_full_size(gcmod, name):
    """The paper's own synthetic graphs at Table II's largest sizes,
    against closed forms rather than the oracle: n = M^2, m = 2(M-1)(2M-1)
    (Table II), T = 4(M-1)^2 (= Table II / 2, reading A9); per edge, a
    horizontal or vertical edge has support 4 (2 on the border row / column it
    runs along), a diagonal edge 2; every triangle uses a diagonal, so the
    4-truss is the whole graph, the 5-truss is empty and every trussness is 4."""
    import torch
    M = gen.CONFIGS[name].n
    u, v = gen.CONFIGS[name].generate()
    c = gcmod.Context(0, torch.cuda.current_stream())
    try:
        c.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
        c.build_csr()
        n, m = c.num_vertices(), c.num_edges()
        T = c.triangle_count()
        sup = c.edge_support()
        cu, cv = c.get_edges()
        m4 = c.ktruss(4)[1]
        m5 = c.ktruss(5)[1]
        tau, kmax = c.truss_decomposition()
    finally:
        c.close()
    assert n == M * M and m == 2 * (M - 1) * (2 * M - 1) and T == 4 * (M - 1) ** 2
    d = cv.astype(np.int64) - cu.astype(np.int64)
    r, col = cu // M, cu % M
    want = np.full(m, 2, np.uint32)
    want[(d == 1) & (r > 0) & (r < M - 1)] = 4
    want[(d == M) & (col > 0) & (col < M - 1)] = 4
    assert np.all((d == 1) | (d == M) | (d == M - 1) | (d == M + 1))
    assert np.array_equal(sup, want)
    assert m4 == m and m5 == 0 and kmax == 4 and np.all(tau == 4)


# ------------------------------------------------------------------ configs --
def test_c1_full(ctx):
    u, v = gen.CONFIGS["C1"].generate()
    g = check_all(ctx, u, v, ks=tuple(range(2, 32)))
    assert ctx.truss_decomposition()[1] >= 3


def test_c2_full(ctx):
    u, v = gen.CONFIGS["C2"].generate()
    check_all(ctx, u, v, ks=(3, 4), decomposition=True)


def load_golden(name):
    """tests/golden/<name>_expected.json, written by scripts/make_golden.py from
    oracle/ only.  A missing file is a failure, not a skip."""
    path = os.path.join(GOLDEN, f"{name.lower()}_expected.json")
    assert os.path.exists(path), f"{path} missing: run `python scripts/make_golden.py {name}`"
    return json.load(open(path))


def hist(a):
    vals, cnt = np.unique(a, return_counts=True)
    return {str(int(x)): int(c) for x, c in zip(vals, cnt)}


def check_trussness_properties(c, d, sup, adj, n_uniform=3000, n_top=500, per_level=1):
    """The decomposition against what holds at any size (tests/truss_props.py):
    the 3-truss mask is {s >= 1} of the golden-checked supports, tau = 2 exactly
    there, tau <= s + 2, kmax = max tau, and on a seeded sample (uniform edges,
    the deepest edges, one edge of every level) the h-index identity
    kappa(e) = H({min(kappa(f), kappa(g))}) - soundness and maximality of every
    level at that edge.  `adj` is the oracle's adjacency
    (rows with edge ids) of the same input."""
    import truss_props as tp
    assert np.array_equal(adj.cu, c.get_edges()[0])
    mask, m_alive = c.ktruss(3)
    assert m_alive == d["m"] - d["support_zero"] and np.array_equal(mask.astype(bool), sup > 0)
    del mask
    tau, kmax = c.truss_decomposition()
    tp.check_global(sup, tau, kmax)
    edges = tp.sample_edges(tau, n_uniform, n_top, per_level, seed=d["m"] % 1000)
    n = tp.check_local(adj.ptr, adj.col, adj.eid, adj.cu, adj.cv, tau, edges)
    assert n >= min(n_uniform // 2, tau.size)
    return tau, kmax


def check_golden(c, d, ks=(3, 4, 5, 6), fused_k=None, adj=None):
    """Every result of one built context against the oracle's golden file:
    canonical edge list, T, supports, k-truss masks, trussness and kmax
    (sha256 of the canonical-order arrays, plus histograms)."""
    import torch
    m = c.num_edges()
    assert (c.num_vertices(), m) == (d["n"], d["m"])
    cu, cv = c.get_edges()
    assert sha(np.stack([cu, cv], axis=1)) == d["canonical_sha256"]
    del cu, cv
    assert c.triangle_count() == d["triangles"]
    sup = c.edge_support()
    assert int(sup.max(initial=0)) == d["support_max"] and int((sup == 0).sum()) == d["support_zero"]
    assert sha(sup) == d["support_sha256"]
    if d.get("trussness_pending"):
        # the golden holds T and supports only (scripts/make_golden.py --support-only): the
        # decomposition is checked by its size-independent properties, then the missing exact
        # comparison is reported as an expected failure
        tau, kmax = check_trussness_properties(c, d, sup, adj)
        part = d.get("trussness_partial")
        if part:
            # O-8 finished every level below clip + 1 before its deadline: min(trussness, clip) is exact
            clip = np.minimum(tau, np.int32(part["clip"])).astype(np.int32)
            assert kmax >= part["kmax_at_least"]
            assert int((tau >= part["clip"]).sum()) == part["live_edges"]
            assert hist(clip) == part["clip_hist"]
            assert sha(clip) == part["clip_sha256"]
            pytest.xfail(f"exact trussness golden only below level {part['clip']} (O-8 stopped at its deadline): "
                         f"{d['m'] - part['live_edges']} of {d['m']} edges exact, the rest by properties "
                         f"(kmax {kmax})")
        pytest.xfail(f"no exact trussness golden for this config (O-8 takes hours); T, every support and the "
                     f"trussness properties hold (kmax {kmax}, {np.unique(tau).size} levels)")
    for k in ks:
        mask, m_alive = c.ktruss(k)
        assert m_alive == d["ktruss_size"][str(k)], k
        assert sha(mask) == d["ktruss_sha256"][str(k)], k
    for fk in (fused_k if isinstance(fused_k, tuple) else () if fused_k is None else (fused_k,)):
        # bench.py's step: the fused call, device outputs
        dsup = torch.empty(m, dtype=torch.int32, device="cuda")
        dmask = torch.empty(m, dtype=torch.uint8, device="cuda")
        T, _, _, m_alive = c.ktruss_analysis(fk, dsup, dmask)
        assert T == d["triangles"] and m_alive == d["ktruss_size"][str(fk)]
        assert sha(dsup.cpu().numpy().view(np.uint32)) == d["support_sha256"]
        assert sha(dmask.cpu().numpy()) == d["ktruss_sha256"][str(fk)]
        del dsup, dmask
    tau, kmax = c.truss_decomposition()
    assert kmax == d["kmax"]
    assert hist(tau) == d["trussness_hist"]
    assert sha(tau.astype(np.int32)) == d["trussness_sha256"]
    for k in (d["kmax"], d["kmax"] + 1):
        assert sha((tau >= k).astype(np.uint8)) == d["ktruss_sha256"][str(k)]


def run_config_golden(gcmod, name, props=False, **kw):
    """Full-size config in bench.py's launch configuration (torch's current
    stream, device-resident raw lists)."""
    import torch
    d = load_golden(name)
    u, v = gen.CONFIGS[name].generate()
    assert u.size == d["nnz"]
    c = gcmod.Context(0, torch.cuda.current_stream())
    try:
        c.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
        adj = oracle.OracleGraph(u, v) if (props or d.get("trussness_pending")) else None
        del u, v
        c.build_csr()
        check_golden(c, d, adj=adj, **kw)
        if props and not d.get("trussness_pending"):   # the checker accepts an exact decomposition at size
            check_trussness_properties(c, d, c.edge_support(), adj)
    finally:
        c.close()


def test_c3_full(gcmod):
    """BASELINE configs[2] (R-MAT s20): T, every support, the k-truss masks at
    k = 3, 4, 5, 6 (O-5, the definition) and the full trussness
    (O-7, equal to O-5's masks as tau >= k) — exact, every edge."""
    run_config_golden(gcmod, "C3", fused_k=4, props=True)


def test_c4_full(gcmod):
    """BASELINE configs[3] (R-MAT s24, the bench workload): T, every support,
    k-truss masks k = 3..6 and the full trussness / kmax against O-3, O-4 and
    O-7 — exact, every edge."""
    run_config_golden(gcmod, "C4", fused_k=(4, 3))   # 4: bench.py's timed call


# ------------------------------------------------------- kernel class forcing --
@pytest.mark.parametrize("force", [0, 1, 2, 3])
def test_forced_classes(ctx, gcmod, force):
    """Every intersection variant, forced over whole graphs."""
    u1, v1 = gen.CONFIGS["C1"].generate()
    u2, v2 = gen.rmat(13, 16, seed=9)
    try:
        ctx.set_option(gcmod.GC_OPT_FORCE_CLASS, force)
        for u, v in [(u1, v1), (u2, v2)]:
            g = oracle.OracleGraph(u, v)
            run_gpu(ctx, u, v)
            assert ctx.triangle_count() == g.triangle_count()
            assert np.array_equal(ctx.edge_support(), g.support())
    finally:
        ctx.set_option(gcmod.GC_OPT_FORCE_CLASS, -1)


@pytest.mark.parametrize("bitmap", [0, 1])
def test_heavy_head_bitmap_and_hash(ctx, gcmod, bitmap):
    """The heavy-head (class 2) kernel in both membership modes, forced on all heads."""
    u, v = gen.rmat(13, 16, seed=19)
    g = oracle.OracleGraph(u, v)
    try:
        ctx.set_option(gcmod.GC_OPT_FORCE_CLASS, 2)
        ctx.set_option(gcmod.GC_OPT_BLOCK_BITMAP, bitmap)
        run_gpu(ctx, u, v)
        assert ctx.triangle_count() == g.triangle_count()
        assert np.array_equal(ctx.edge_support(), g.support())
        for chunk in (32, 777):
            ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, chunk)
            assert ctx.triangle_count() == g.triangle_count()
            assert np.array_equal(ctx.edge_support(), g.support())
    finally:
        ctx.set_option(gcmod.GC_OPT_FORCE_CLASS, -1)
        ctx.set_option(gcmod.GC_OPT_BLOCK_BITMAP, 1)
        ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, 32768)


@pytest.mark.parametrize("huge_max", [0, 40, 8192])
def test_huge_head_hash_and_global_probe(ctx, gcmod, huge_max):
    """The huge-head (class 3) block kernel forced on all heads: shared hash
    (d+ <= huge_max) and global binary search (d+ > huge_max), with small and
    default task chunks (several block tasks per head, exact wedge split)."""
    u, v = gen.rmat(13, 16, seed=23)
    g = oracle.OracleGraph(u, v)
    try:
        ctx.set_option(gcmod.GC_OPT_FORCE_CLASS, 3)
        ctx.set_option(gcmod.GC_OPT_HUGE_MAX, huge_max)
        run_gpu(ctx, u, v)
        for chunk in (4096, 57):
            ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, chunk)
            assert ctx.triangle_count() == g.triangle_count()
            assert np.array_equal(ctx.edge_support(), g.support())
            want, _ = g.ktruss(4)
            assert np.array_equal(ctx.ktruss(4)[0], want)
    finally:
        ctx.set_option(gcmod.GC_OPT_FORCE_CLASS, -1)
        ctx.set_option(gcmod.GC_OPT_HUGE_MAX, 8192)
        ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, 32768)


def test_task_chunk_sizes(ctx, gcmod):
    u, v = gen.rmat(12, 16, seed=13)
    g = oracle.OracleGraph(u, v)
    want = g.support()
    try:
        for chunk in (32, 100, 1000, 1 << 20):
            ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, chunk)
            run_gpu(ctx, u, v)
            assert np.array_equal(ctx.edge_support(), want)
    finally:
        ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, 32768)


def test_wide_bitmap_class(ctx, gcmod):
    """Class 4 (4096 < d+ <= 8192, N+(v) inside the rank window: the bitmap
    kernel with 8192 (v,w) counters) on a dense G(5000, 0.85): supports
    against dense A^2 on the edges (P5), T = trace(A^3)/6, default and small
    task chunks (a head split over several block tasks)."""
    rng = np.random.default_rng(41)
    n = 5000
    u, v = random_graph(n, 0.85, rng)
    A = np.zeros((n, n))
    A[u, v] = 1
    A[v, u] = 1
    A2 = A @ A                                   # exact in float64 (entries < 2^53)
    try:
        for chunk in (32768, 2000):
            ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, chunk)
            run_gpu(ctx, u, v)
            assert ctx.stats()["tasks"][4] > 0
            cu, cv = ctx.get_edges()
            sup = ctx.edge_support()
            assert np.array_equal(sup, A2[cu, cv].astype(np.uint32))
            assert ctx.triangle_count() == int(round(np.trace(A2 @ A))) // 6
    finally:
        ctx.set_option(gcmod.GC_OPT_TASK_CHUNK, 32768)


def test_large_clique_all_classes(ctx):
    """K_4200: out-degrees span the classes up to the wide-bitmap one (4)."""
    n = 4200
    iu, ju = np.triu_indices(n, 1)
    run_gpu(ctx, iu.astype(np.int32), ju.astype(np.int32))
    assert ctx.triangle_count() == math.comb(n, 3)
    assert np.all(ctx.edge_support() == n - 2)


# -------------------------------------------------- loopback partitions (T3) --
@pytest.mark.parametrize("parts", [2, 3, 8])
def test_loopback_partitions(gcmod, parts):
    u, v = gen.rmat(13, 16, seed=17)
    g = oracle.OracleGraph(u, v)
    with gcmod.Context(0) as c:
        c.comm_init_loopback(parts)
        c.load_edges(u, v)
        c.build_csr()
        assert c.triangle_count() == g.triangle_count()
        assert np.array_equal(c.edge_support(), g.support())
        for k in (3, 5, 7):
            want, _ = g.ktruss(k)
            assert np.array_equal(c.ktruss(k)[0], want), k
        tau, kmax = c.truss_decomposition()
        want_tau, want_kmax = g.truss_decomposition()
        assert np.array_equal(tau, want_tau) and kmax == want_kmax


@pytest.mark.parametrize("compact", [0, 2, 3, 5, 8])
def test_decomposition_row_compaction(gcmod, compact):
    """Peeler with dead-entry compaction of the adjacency rows off (0) or each
    time the live edges fall to (v-1)/v of the last compaction (v = 2: every
    halving; 5: the decomposition default, 4/5) — C1 decomposition and
    k-truss, R-MAT s12."""
    for u, v in [gen.CONFIGS["C1"].generate(), gen.rmat(12, 16, seed=29)]:
        g = oracle.OracleGraph(u, v)
        with gcmod.Context(0) as c:
            c.set_option(gcmod.GC_OPT_COMPACT, compact)
            c.load_edges(u, v)
            c.build_csr()
            for k in (5, 9):
                want, _ = g.ktruss(k)
                assert np.array_equal(c.ktruss(k)[0], want), k
            tau, kmax = c.truss_decomposition()
            want_tau, want_kmax = g.truss_decomposition()
            assert np.array_equal(tau, want_tau) and kmax == want_kmax
            if compact:
                assert c.stats()["compactions"] > 0
            # a second call after compaction starts from refilled rows
            want, _ = g.ktruss(4)
            assert np.array_equal(c.ktruss(4)[0], want)


@pytest.mark.parametrize("heavy", [1, 16])
def test_grouped_dense_core_rounds(gcmod, heavy):
    """Every peel round grouped (heavy edges by pivot, staged as a shared
    bitmap; light ones by the per-edge search): k-truss and decomposition of
    C1, an R-MAT s12 and a 300-clique with a pendant fan, against the oracle."""
    q = np.arange(300, dtype=np.int32)
    a, b = np.triu_indices(q.size, 1)
    fan = np.arange(300, 700, dtype=np.int32)
    graphs = [gen.CONFIGS["C1"].generate(), gen.rmat(12, 16, seed=31),
              (np.concatenate([q[a], fan, fan[1:]]), np.concatenate([q[b], fan % 7, fan[:-1]]))]
    for u, v in graphs:
        g = oracle.OracleGraph(u, v)
        for compact in (0, 2):
            with gcmod.Context(0) as c:
                c.set_option(gcmod.GC_OPT_GROUP_PEEL, 1)
                c.set_option(gcmod.GC_OPT_GROUP_HEAVY, heavy)
                c.set_option(gcmod.GC_OPT_COMPACT, compact)
                c.load_edges(u, v)
                c.build_csr()
                for k in (4, 7):
                    want, _ = g.ktruss(k)
                    assert np.array_equal(c.ktruss(k)[0], want), k
                tau, kmax = c.truss_decomposition()
                want_tau, want_kmax = g.truss_decomposition()
                assert np.array_equal(tau, want_tau) and kmax == want_kmax


def test_peel_register_builds(gcmod, monkeypatch):
    """Both register budgets of the peel kernel (GC_PEEL_BIG=1: the 64-register
    build for every round; default: the 32-register build) give the oracle's
    k-trusses and decomposition on C1 and an R-MAT s12."""
    for env in ("1", None):
        if env:
            monkeypatch.setenv("GC_PEEL_BIG", env)
        else:
            monkeypatch.delenv("GC_PEEL_BIG", raising=False)
        for u, v in [gen.CONFIGS["C1"].generate(), gen.rmat(12, 16, seed=61)]:
            g = oracle.OracleGraph(u, v)
            with gcmod.Context(0) as c:
                c.load_edges(u, v)
                c.build_csr()
                for k in (4, 6):
                    want, _ = g.ktruss(k)
                    assert np.array_equal(c.ktruss(k)[0], want), (env, k)
                tau, kmax = c.truss_decomposition()
                want_tau, want_kmax = g.truss_decomposition()
                assert np.array_equal(tau, want_tau) and kmax == want_kmax, env


@pytest.mark.parametrize("parts", [1, 2, 5])
def test_partitioned_peeler_c1_and_fixtures(gcmod, parts):
    """The multi-GPU peeler (removed-edge bitmap per round, owner-only
    decrements): P = 1 through GC_OPT_PEEL_PART, P > 1 as
    loopback virtual ranks with one support copy each.  Includes the A5
    tie-break fixture, whose two simultaneous removals share a triangle."""
    cases = [gen.CONFIGS["C1"].generate()]
    d = json.load(open(os.path.join(GOLDEN, "k4_ear.json")))
    cases.append((np.array(d["raw_u"], np.int32), np.array(d["raw_v"], np.int32)))
    cases.append(random_graph(90, 0.3, np.random.default_rng(parts)))
    for u, v in cases:
        g = oracle.OracleGraph(u, v)
        with gcmod.Context(0) as c:
            if parts == 1:
                c.set_option(gcmod.GC_OPT_PEEL_PART, 1)
            else:
                c.comm_init_loopback(parts)
            c.load_edges(u, v)
            c.build_csr()
            for k in (3, 4, 6):
                want, _ = g.ktruss(k)
                mask, m_alive = c.ktruss(k)
                assert np.array_equal(mask, want) and m_alive == int(want.sum()), k
            tau, kmax = c.truss_decomposition()
            want_tau, want_kmax = g.truss_decomposition()
            assert np.array_equal(tau, want_tau) and kmax == want_kmax


# ------------------------------------------------------- triangle listing ----
def _brute_triangles(g):
    """Independent listing from the oracle's canonical edges: {a<b<w} with all three edges present."""
    adj = {}
    for a, b in zip(g.cu.tolist(), g.cv.tolist()):
        adj.setdefault(a, set()).add(b)
        adj.setdefault(b, set()).add(a)
    out = set()
    for a, b in zip(g.cu.tolist(), g.cv.tolist()):
        for w in adj[a] & adj[b]:
            if w > b:
                out.add((a, b, w))
    return out


def test_list_triangles(gcmod, ctx):
    """gc_list_triangles (Alg. 1's triangle records): the same set as
    an independent enumeration, each triangle once, ids ascending in a row;
    the king grid's triangles all sit inside 2x2 pixel cells."""
    for u, v in [gen.CONFIGS["C1"].generate(), gen.rmat(11, 16, seed=43), random_graph(70, 0.3, np.random.default_rng(9))]:
        g = oracle.OracleGraph(u, v)
        run_gpu(ctx, u, v)
        tri = ctx.list_triangles()
        assert tri.shape == (g.triangle_count(), 3)
        assert np.all(tri[:, 0] < tri[:, 1]) and np.all(tri[:, 1] < tri[:, 2])
        got = set(map(tuple, tri.tolist()))
        assert len(got) == len(tri) and got == _brute_triangles(g)
    M = 64
    u, v = gen.king_grid(M)
    run_gpu(ctx, u, v)
    tri = ctx.list_triangles()
    assert len(tri) == 4 * (M - 1) ** 2
    r, c = tri // M, tri % M
    assert np.all(r.max(1) - r.min(1) == 1) and np.all(c.max(1) - c.min(1) == 1)
    with pytest.raises(gcmod.GcError) as e:
        ctx.list_triangles(capacity=10)
    assert e.value.code == gcmod.GC_ERR_RANGE


# ------------------------------------------------ fused analysis entry point --
@pytest.mark.parametrize("parts", [0, 3])
def test_ktruss_analysis_one_pass(gcmod, parts):
    """gc_ktruss_analysis: triangle count, supports and k-truss mask from one
    support pass equal the oracle's (and the separate calls'); NULL outputs."""
    import ctypes
    cases = [gen.CONFIGS["C1"].generate(), gen.rmat(12, 16, seed=41), random_graph(60, 0.4, np.random.default_rng(3))]
    for u, v in cases:
        g = oracle.OracleGraph(u, v)
        with gcmod.Context(0) as c:
            if parts:
                c.comm_init_loopback(parts)
            c.load_edges(u, v)
            c.build_csr()
            for k in (2, 3, 5):
                T, sup, mask, m_alive = c.ktruss_analysis(k)
                want, _ = g.ktruss(k)
                assert T == g.triangle_count() and np.array_equal(sup, g.support())
                assert np.array_equal(mask, want) and m_alive == int(want.sum())
            # only the count / only the mask
            t = ctypes.c_uint64()
            rc = gcmod.load_library().gc_ktruss_analysis(c._h, 4, ctypes.byref(t), None, None, None)
            assert rc == 0 and t.value == g.triangle_count()
            mk = np.empty(g.m, np.uint8)
            rc = gcmod.load_library().gc_ktruss_analysis(c._h, 4, None, None, mk.ctypes.data, None)
            assert rc == 0 and np.array_equal(mk, g.ktruss(4)[0])
            with pytest.raises(gcmod.GcError):
                c.ktruss_analysis(1)


# --------------------------------------------------- API / pointer kinds ----
def test_staged_edges(gcmod):
    """gc_stage_edges: the next graph's copy is enqueued while the current one
    stays usable; the next build consumes it.  Host (pageable and pinned) and
    device sources, staging as the first call, a replaced stage, and a stage
    discarded by gc_load_edges, all against the oracle."""
    import torch
    ga = gen.rmat(11, 16, seed=41)
    gb = gen.rmat(12, 8, seed=42)
    gcx = gen.rmat(10, 16, seed=43)
    oa, ob, oc = (oracle.OracleGraph(*g) for g in (ga, gb, gcx))
    with gcmod.Context(0) as c:
        c.stage_edges(*ga)                                    # first call: stage, then build
        c.build_csr()
        assert c.triangle_count() == oa.triangle_count()
        pu = torch.from_numpy(gb[0]).pin_memory()
        pv = torch.from_numpy(gb[1]).pin_memory()
        c.stage_edges(pu, pv)                                 # graph A stays valid meanwhile
        assert np.array_equal(c.edge_support(), oa.support())
        cu, cv = c.get_edges()
        assert np.array_equal(cu, oa.cu) and np.array_equal(cv, oa.cv)
        c.build_csr()
        assert c.triangle_count() == ob.triangle_count()
        assert np.array_equal(c.edge_support(), ob.support())
        c.stage_edges(*ga)                                    # replaced before use
        c.stage_edges(torch.from_numpy(gcx[0]).cuda(), torch.from_numpy(gcx[1]).cuda())
        c.build_csr()
        assert np.array_equal(c.edge_support(), oc.support())
        want, _ = oc.ktruss(4)
        assert np.array_equal(c.ktruss(4)[0], want)
        c.stage_edges(*gb)                                    # discarded by gc_load_edges
        c.load_edges(*ga)
        c.build_csr()
        assert c.triangle_count() == oa.triangle_count()
        c.stage_edges(np.zeros(0, np.int32), np.zeros(0, np.int32))   # empty graph
        c.build_csr()
        assert c.num_edges() == 0 and c.triangle_count() == 0


def test_async_outputs(gcmod):
    """gc_ktruss_analysis_async: scalars at return, per-edge outputs after
    gc_wait; pipelined with gc_stage_edges; a following synchronous call
    waits for the pending read-back before reusing its staging buffers."""
    import torch
    ga = gen.rmat(12, 16, seed=51)
    gb = gen.rmat(11, 8, seed=52)
    oa, ob = oracle.OracleGraph(*ga), oracle.OracleGraph(*gb)
    with gcmod.Context(0) as c:
        c.load_edges(*ga)
        c.build_csr()
        m = c.num_edges()
        hs = torch.empty(m, dtype=torch.int32).pin_memory()
        hm = torch.empty(m, dtype=torch.uint8).pin_memory()
        T, ma = c.ktruss_analysis_async(4, hs, hm)
        want, _ = oa.ktruss(4)
        assert T == oa.triangle_count() and ma == int(want.sum())
        c.stage_edges(*gb)                          # next graph's copy while the read-back runs
        sup_sync = c.edge_support()                 # waits for the pending read-back first
        c.wait()
        assert np.array_equal(hs.numpy().view(np.uint32), oa.support()) and np.array_equal(hm.numpy(), want)
        assert np.array_equal(sup_sync, oa.support())
        c.build_csr()
        mb = c.num_edges()
        ds = torch.empty(mb, dtype=torch.int32, device="cuda")
        dm = torch.empty(mb, dtype=torch.uint8, device="cuda")
        T, ma = c.ktruss_analysis_async(3, ds, dm)  # device outputs
        c.wait()
        want, _ = ob.ktruss(3)
        assert T == ob.triangle_count() and ma == int(want.sum())
        assert np.array_equal(ds.cpu().numpy().view(np.uint32), ob.support())
        assert np.array_equal(dm.cpu().numpy(), want)


def test_device_pointers_and_determinism(ctx):
    import torch
    u, v = gen.rmat(12, 16, seed=21)
    g = oracle.OracleGraph(u, v)
    du = torch.from_numpy(u).cuda()
    dv = torch.from_numpy(v).cuda()
    ctx.load_edges(du, dv)
    ctx.build_csr()
    m = ctx.num_edges()
    out = torch.empty(m, dtype=torch.int32, device="cuda")
    ctx.edge_support(out.view(torch.int32))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), g.support())
    first = ctx.edge_support()
    for _ in range(3):
        assert np.array_equal(ctx.edge_support(), first)
        assert ctx.triangle_count() == g.triangle_count()


def test_errors(ctx, gcmod):
    with pytest.raises(gcmod.GcError) as e:
        run_gpu(ctx, np.array([0, -1], np.int32), np.array([1, 2], np.int32))
    assert e.value.code == gcmod.GC_ERR_INVALID
    run_gpu(ctx, np.array([0, 1], np.int32), np.array([1, 2], np.int32))
    with pytest.raises(gcmod.GcError) as e:
        ctx.ktruss(1)
    assert e.value.code == gcmod.GC_ERR_INVALID
    with gcmod.Context(0) as c2:
        with pytest.raises(gcmod.GcError) as e:
            c2.triangle_count()
        assert e.value.code == gcmod.GC_ERR_STATE
        c2.wait()                                            # nothing pending: a no-op
        with pytest.raises(gcmod.GcError) as e:              # NULL source with nnz > 0
            c2._check(c2._L.gc_stage_edges(c2._h, None, None, 5))
        assert e.value.code == gcmod.GC_ERR_INVALID
        with pytest.raises(gcmod.GcError) as e:              # staged, not built yet
            c2.stage_edges(np.array([0, 1], np.int32), np.array([1, 2], np.int32))
            c2.num_edges()
        assert e.value.code == gcmod.GC_ERR_STATE
        c2.build_csr()
        assert c2.num_edges() == 2
        with pytest.raises(gcmod.GcError) as e:
            c2.ktruss_analysis_async(1, np.empty(2, np.uint32), np.empty(2, np.uint8))
        assert e.value.code == gcmod.GC_ERR_INVALID


# ------------------------------------------- k-truss byte-model terms (§8(d)) --
def test_work_stats_match_oracle_replay(gcmod):
    """GC_OPT_WORK_STATS: the peeler's Σ min(d(a), d(b)) over frontier edges
    with support > 0 and its decrement count D equal the oracle's batch
    replay (O-5 / O-6 with work=True) for single k-trusses and whole
    decompositions — the terms bench.py's k-truss roofline is built from."""
    cases = [gen.CONFIGS["C1"].generate(), gen.rmat(12, 16, seed=71)]
    for f in ("k4_ear.json", "hub_two_k4.json"):
        d = json.load(open(os.path.join(GOLDEN, f)))
        cases.append((np.array(d["raw_u"], np.int32), np.array(d["raw_v"], np.int32)))
    for u, v in cases:
        g = oracle.OracleGraph(u, v)
        with gcmod.Context(0) as c:
            c.set_option(gcmod.GC_OPT_WORK_STATS, 1)
            c.load_edges(u, v)
            c.build_csr()
            for k in (3, 4, 5, 7):
                want_mask, _, w = g.ktruss(k, work=True)
                T, _, mask, _ = c.ktruss_analysis(k)
                st = c.stats()
                assert np.array_equal(mask, want_mask), k
                assert (st["peel_sum_min"], st["peel_decrements"]) == (w["sum_min"], w["decrements"]), k
            tau, kmax = c.truss_decomposition()
            want_tau, want_kmax, w = g.truss_decomposition(work=True)
            st = c.stats()
            assert np.array_equal(tau, want_tau) and kmax == want_kmax
            assert (st["peel_sum_min"], st["peel_decrements"]) == (w["sum_min"], w["decrements"])


# ------------------------------------------------- NCCL on the hardware (§8(e)) --
def test_nccl_one_rank_communicator(gcmod):
    """A real one-rank NCCL communicator (gc_comm_init, nranks = 1; NCCL resolved
    by dlopen): the triangle count and support passes end in ncclAllReduce, the
    peeler is the partitioned one (removed-edge bitmap per round through the
    in-place ncclAllGather, zero-support bitmap and ncclAllReduce(min) at each
    level start) — results equal the oracle's."""
    cases = [gen.CONFIGS["C1"].generate(), gen.rmat(12, 16, seed=81)]
    d = json.load(open(os.path.join(GOLDEN, "k4_ear.json")))
    cases.append((np.array(d["raw_u"], np.int32), np.array(d["raw_v"], np.int32)))
    for u, v in cases:
        g = oracle.OracleGraph(u, v)
        with gcmod.Context(0) as c:
            c.comm_init(gcmod.nccl_unique_id(), 1, 0)
            c.load_edges(u, v)
            c.build_csr()
            assert c.triangle_count() == g.triangle_count()
            assert np.array_equal(c.edge_support(), g.support())
            for k in (3, 4, 6):
                want, _ = g.ktruss(k)
                mask, m_alive = c.ktruss(k)
                assert np.array_equal(mask, want) and m_alive == int(want.sum()), k
            T, sup, mask, _ = c.ktruss_analysis(5)
            assert T == g.triangle_count() and np.array_equal(mask, g.ktruss(5)[0])
            tau, kmax = c.truss_decomposition()
            want_tau, want_kmax = g.truss_decomposition()
            assert np.array_equal(tau, want_tau) and kmax == want_kmax
            assert c.stats()["peel_rounds"] > 0 or want_kmax <= 3



@pytest.mark.parametrize("setup", ["part1", "loop2", "loop3", "loop8", "nccl1"])
def test_partitioned_build(gcmod, setup):
    """gc_build_csr across owners (GC_OPT_BUILD_PART): each
    owner sorts the raw pairs of its low-endpoint id range, the oriented edges
    of its tail-rank range and the in-edges of its head-rank range; the parts
    are concatenated (NCCL: grouped broadcasts).  One owner forced, loopback
    2 / 3 / 8 virtual ranks, and a real one-rank NCCL communicator: canonical
    list, supports, k-truss and decomposition equal the oracle's, on graphs
    with duplicates, reversed pairs, self loops, a hub and degenerate inputs."""
    rng = np.random.default_rng(90)
    hub_u = np.zeros(3000, np.int32)
    hub_v = rng.integers(1, 5000, 3000).astype(np.int32)
    cases = [gen.CONFIGS["C1"].generate(), gen.rmat(13, 16, seed=91), (hub_u, hub_v),
             (np.array([5, 5, 2, 9, 2], np.int32), np.array([5, 2, 5, 1 << 20, 2], np.int32)),
             (np.array([3, 3], np.int32), np.array([3, 3], np.int32)),
             (np.zeros(0, np.int32), np.zeros(0, np.int32))]
    for u, v in cases:
        g = oracle.OracleGraph(u, v)
        with gcmod.Context(0) as c:
            if setup.startswith("loop"):
                c.comm_init_loopback(int(setup[4:]))
            elif setup == "nccl1":
                c.comm_init(gcmod.nccl_unique_id(), 1, 0)
            c.set_option(gcmod.GC_OPT_BUILD_PART, 1)
            c.load_edges(u, v)
            c.build_csr()
            assert (c.num_vertices(), c.num_edges()) == (g.n, g.m)
            cu, cv = c.get_edges()
            assert np.array_equal(cu, g.cu) and np.array_equal(cv, g.cv)
            assert c.triangle_count() == g.triangle_count()
            assert np.array_equal(c.edge_support(), g.support())
            want, _ = g.ktruss(4)
            assert np.array_equal(c.ktruss(4)[0], want)
            tau, kmax = c.truss_decomposition()
            want_tau, want_kmax = g.truss_decomposition()
            assert np.array_equal(tau, want_tau) and kmax == want_kmax


# Last in the file (the -x run stops at a failure): the largest config.
def test_c5_full(gcmod):
    """BASELINE configs[4] (skewed R-MAT s26, ~9.3e8 edges, int64 offsets) on
    one GPU: T, every support and the full truss decomposition (trussness of
    every edge, kmax) against O-3 (T = sum of supports / 3, P4) and O-8 —
    exact."""
    run_config_golden(gcmod, "C5", ks=(3,))
