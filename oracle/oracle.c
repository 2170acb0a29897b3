/*
 * oracle.c — CPU ORACLE for per-edge triangle support, triangle count and
 * k-truss (Samsi et al., "Static Graph Challenge: Subgraph Isomorphism",
 * arXiv 1708.06866; cited as P:<line> of PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  The
 * product path (paper_1708_06866_b200/, libgc.so) never links, loads or
 * calls it, and this file shares no code, header, table or constant with it.
 *
 * Plain, slow and obviously correct: each function writes out a definition
 * from the paper (or, where the paper gives an array algorithm, its
 * element-wise meaning) with no blocking or reordering beyond it.  Integer
 * results are independent of the thread count (threads take static chunks
 * of independent edges and only write their own outputs).
 *
 *   O-1  or_canonicalize      self loops removed, reverse edges added,
 *                             duplicates dropped (reading A1)
 *   O-2  or_adjacency         N(x) sorted ascending, with edge ids
 *   O-3  or_support           support(a,b) = |N(a) ∩ N(b)|  (P:283-288:
 *                             "the overlap of the neighborhoods")
 *   O-4  or_triangle_count    #{a<b<w pairwise adjacent}
 *   O-5  or_ktruss            Alg. 4 batch semantics: repeat
 *                             { recompute s on the alive subgraph;
 *                               x = {s < k-2}; drop x } until x is empty
 *   O-6  or_truss_decomposition  P:299-302: k = 3, 4, ... each from the
 *                             previous result until empty
 *   O-7  or_truss_sequential  tier 2: one-edge-at-a-time min-support peel
 *                             (bucket order); equal to O-6 by uniqueness
 *                             of the maximal k-truss (reading A2/A8)
 *   O-8  or_truss_parallel    tier 2: Alg. 4's incremental update
 *                             element-wise, rounds in parallel
 *                             over the edges of x; equal to O-6 and O-7
 *
 * Pins: tests/test_oracle_pins.py (brute force, closed forms, trace(A^3)/6,
 * literal Alg. 1-4 in scipy, networkx, Table II, invariants).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>
#include <stdio.h>
#include <time.h>

static int n_threads(int t) {
    if (t > 0) return t;
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    if (c < 1) c = 1;
    if (c > 256) c = 256;
    return (int)c;
}

/* Run fn(ctx, i0, i1, t) over [0, N) in T static chunks (chunk t). */
typedef void (*range_fn)(void* ctx, int64_t i0, int64_t i1, int t);
typedef struct { range_fn fn; void* ctx; int64_t i0, i1; int t; } range_job;
static void* range_tramp(void* a) { range_job* j = (range_job*)a; j->fn(j->ctx, j->i0, j->i1, j->t); return NULL; }
static void parallel_for(int64_t N, int T, range_fn fn, void* ctx) {
    T = n_threads(T);
    if (N < 1024 || T == 1) { fn(ctx, 0, N, 0); return; }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * T);
    range_job* jb = (range_job*)malloc(sizeof(range_job) * T);
    for (int t = 0; t < T; ++t) {
        jb[t].fn = fn; jb[t].ctx = ctx; jb[t].i0 = N * t / T; jb[t].i1 = N * (t + 1) / T; jb[t].t = t;
        pthread_create(&th[t], NULL, range_tramp, &jb[t]);
    }
    for (int t = 0; t < T; ++t) pthread_join(th[t], NULL);
    free(th); free(jb);
}

/* Run fn over [0, N) in chunks of `grain` taken from a shared counter by T
 * threads (for uneven per-item work; results must not depend on who runs
 * which chunk). */
typedef struct { range_fn fn; void* ctx; int64_t N, grain; int64_t* next; int t; } dyn_job;
static void* dyn_tramp(void* a) {
    dyn_job* j = (dyn_job*)a;
    for (;;) {
        const int64_t i0 = __atomic_fetch_add(j->next, j->grain, __ATOMIC_RELAXED);
        if (i0 >= j->N) break;
        j->fn(j->ctx, i0, i0 + j->grain < j->N ? i0 + j->grain : j->N, j->t);
    }
    return NULL;
}
static void parallel_for_dynamic(int64_t N, int T, int64_t grain, range_fn fn, void* ctx) {
    T = n_threads(T);
    if (N <= grain || T == 1) { fn(ctx, 0, N, 0); return; }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * T);
    dyn_job* jb = (dyn_job*)malloc(sizeof(dyn_job) * T);
    int64_t next = 0;
    for (int t = 0; t < T; ++t) {
        jb[t].fn = fn; jb[t].ctx = ctx; jb[t].N = N; jb[t].grain = grain; jb[t].next = &next; jb[t].t = t;
        pthread_create(&th[t], NULL, dyn_tramp, &jb[t]);
    }
    for (int t = 0; t < T; ++t) pthread_join(th[t], NULL);
    free(th); free(jb);
}

/* ------------------------------------------------------------ sorting --
 * LSD radix sort of uint64 keys, one byte per pass (a library-primitive
 * sort; pinned against numpy.sort in the tests). */
int or_sort_u64(uint64_t* keys, int64_t N) {
    if (N <= 1) return 0;
    uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)N);
    if (!tmp) return -1;
    uint64_t* src = keys; uint64_t* dst = tmp;
    for (int pass = 0; pass < 8; ++pass) {
        int sh = 8 * pass;
        int64_t cnt[256];
        memset(cnt, 0, sizeof(cnt));
        for (int64_t i = 0; i < N; ++i) cnt[(src[i] >> sh) & 0xFF]++;
        if (cnt[(src[0] >> sh) & 0xFF] == N) continue;   /* byte constant: pass is identity */
        int64_t off = 0;
        for (int d = 0; d < 256; ++d) { int64_t c = cnt[d]; cnt[d] = off; off += c; }
        for (int64_t i = 0; i < N; ++i) dst[cnt[(src[i] >> sh) & 0xFF]++] = src[i];
        uint64_t* t = src; src = dst; dst = t;
    }
    if (src != keys) memcpy(keys, src, sizeof(uint64_t) * (size_t)N);
    free(tmp);
    return 0;
}

/* ------------------------------------------------------------------ O-1 --
 * Canonical edge list (SURVEY §8(b) "Edge order / ids"):
 * drop u == v, orient (min, max), sort lexicographically, drop duplicates.
 * Edge id = position.  n = max raw id + 1 (0 if nnz == 0).
 * cu, cv: capacity nnz.  Returns m, or -1 on a negative id / OOM. */
int64_t or_canonicalize(const int32_t* u, const int32_t* v, int64_t nnz,
                        int32_t* cu, int32_t* cv, int64_t* n_out) {
    int64_t maxid = -1;
    for (int64_t i = 0; i < nnz; ++i) {
        if (u[i] < 0 || v[i] < 0) return -1;
        if (u[i] > maxid) maxid = u[i];
        if (v[i] > maxid) maxid = v[i];
    }
    *n_out = maxid + 1;
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nnz > 0 ? nnz : 1));
    if (!keys) return -1;
    int64_t k = 0;
    for (int64_t i = 0; i < nnz; ++i) {
        if (u[i] == v[i]) continue;                            /* self loop removed */
        uint32_t a = (uint32_t)(u[i] < v[i] ? u[i] : v[i]);    /* both orientations -> one */
        uint32_t b = (uint32_t)(u[i] < v[i] ? v[i] : u[i]);
        keys[k++] = ((uint64_t)a << 32) | b;
    }
    if (or_sort_u64(keys, k) != 0) { free(keys); return -1; }
    int64_t m = 0;
    for (int64_t i = 0; i < k; ++i) {
        if (i > 0 && keys[i] == keys[i - 1]) continue;         /* duplicate dropped */
        cu[m] = (int32_t)(keys[i] >> 32);
        cv[m] = (int32_t)(keys[i] & 0xFFFFFFFFULL);
        ++m;
    }
    free(keys);
    return m;
}

/* ------------------------------------------------------------------ O-2 --
 * Symmetric adjacency: row x lists N(x) ascending with the canonical id of
 * each edge.  Filling rows while scanning the lexicographic edge list puts
 * lower neighbours (edges (w,x), w<x) before upper ones (edges (x,w), x<w),
 * each ascending, so rows come out sorted.
 * ptr: n+1, col/eid: 2m. */
void or_adjacency(int64_t n, int64_t m, const int32_t* cu, const int32_t* cv,
                  int64_t* ptr, int32_t* col, int32_t* eid) {
    for (int64_t x = 0; x <= n; ++x) ptr[x] = 0;
    for (int64_t e = 0; e < m; ++e) { ptr[cu[e] + 1]++; ptr[cv[e] + 1]++; }
    for (int64_t x = 0; x < n; ++x) ptr[x + 1] += ptr[x];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t x = 0; x < n; ++x) fill[x] = ptr[x];
    for (int64_t e = 0; e < m; ++e) {
        int32_t a = cu[e], b = cv[e];
        col[fill[a]] = b; eid[fill[a]] = (int32_t)e; fill[a]++;
        col[fill[b]] = a; eid[fill[b]] = (int32_t)e; fill[b]++;
    }
    free(fill);
}

/* Sorted-list intersection |A ∩ B| by two-pointer merge; when one list is at
 * least 32x longer, each element of the short list is located in the long
 * one by binary search instead (same set, fewer steps). */
static int64_t lower_bound32(const int32_t* a, int64_t lo, int64_t hi, int32_t x) {
    while (lo < hi) { int64_t mid = lo + (hi - lo) / 2; if (a[mid] < x) lo = mid + 1; else hi = mid; }
    return lo;
}

/* First index in [lo, hi) with a[index] >= x, by exponential then binary
 * search from lo (galloping: log of the distance moved). */
static int64_t gallop32(const int32_t* a, int64_t lo, int64_t hi, int32_t x) {
    int64_t prev = lo, step = 1;
    while (lo < hi && a[lo] < x) { prev = lo + 1; lo += step; step <<= 1; }
    if (lo > hi) lo = hi;
    return lower_bound32(a, prev, lo, x);
}

static int64_t intersect_count(const int32_t* A, int64_t na, const int32_t* B, int64_t nb) {
    if (na == 0 || nb == 0) return 0;
    if (na > nb) { const int32_t* t = A; A = B; B = t; int64_t tn = na; na = nb; nb = tn; }
    int64_t c = 0;
    if (nb >= 32 * na) {
        int64_t lo = 0;
        for (int64_t i = 0; i < na; ++i) {
            lo = lower_bound32(B, lo, nb, A[i]);
            if (lo < nb && B[lo] == A[i]) { ++c; ++lo; }
        }
        return c;
    }
    int64_t i = 0, j = 0;
    while (i < na && j < nb) {
        if (A[i] < B[j]) ++i;
        else if (A[i] > B[j]) ++j;
        else { ++c; ++i; ++j; }
    }
    return c;
}

/* ------------------------------------------------------------------ O-3 --
 * support(a_i, b_i) = |N(a_i) ∩ N(b_i)| for a list of vertex pairs (the
 * canonical edge list, or a sample of it).  sup: npairs. */
typedef struct { const int64_t* ptr; const int32_t* col; const int32_t* a; const int32_t* b; uint32_t* sup; } sup_ctx;
static void sup_range(void* c, int64_t i0, int64_t i1, int t) {
    (void)t;
    sup_ctx* C = (sup_ctx*)c;
    for (int64_t i = i0; i < i1; ++i) {
        int32_t a = C->a[i], b = C->b[i];
        C->sup[i] = (uint32_t)intersect_count(C->col + C->ptr[a], C->ptr[a + 1] - C->ptr[a],
                                              C->col + C->ptr[b], C->ptr[b + 1] - C->ptr[b]);
    }
}
void or_support(const int64_t* ptr, const int32_t* col, int64_t npairs,
                const int32_t* a, const int32_t* b, uint32_t* sup, int nthreads) {
    sup_ctx C = {ptr, col, a, b, sup};
    parallel_for(npairs, nthreads, sup_range, &C);
}

/* ------------------------------------------------------------------ O-4 --
 * Triangle count in vertex-id order: each triangle {a<b<w} is counted once,
 * from its edge (a,b), as a common neighbour w > b (P:159-160 definition).
 * Independent of any degree orientation. */
typedef struct { const int64_t* ptr; const int32_t* col; const int32_t* cu; const int32_t* cv; uint64_t* part; } tc_ctx;
static void tc_range(void* c, int64_t i0, int64_t i1, int t) {
    tc_ctx* C = (tc_ctx*)c;
    uint64_t s = 0;
    for (int64_t e = i0; e < i1; ++e) {
        int32_t a = C->cu[e], b = C->cv[e];
        int64_t a0 = C->ptr[a], a1 = C->ptr[a + 1], b0 = C->ptr[b], b1 = C->ptr[b + 1];
        int64_t pa = lower_bound32(C->col, a0, a1, b + 1);       /* w > b in N(a) */
        int64_t pb = lower_bound32(C->col, b0, b1, b + 1);       /* w > b in N(b) */
        s += (uint64_t)intersect_count(C->col + pa, a1 - pa, C->col + pb, b1 - pb);
    }
    C->part[t] = s;
}
uint64_t or_triangle_count(const int64_t* ptr, const int32_t* col, int64_t m,
                           const int32_t* cu, const int32_t* cv, int nthreads) {
    int T = n_threads(nthreads);
    uint64_t* part = (uint64_t*)calloc((size_t)T + 1, sizeof(uint64_t));
    tc_ctx C = {ptr, col, cu, cv, part};
    parallel_for(m, T, tc_range, &C);
    uint64_t s = 0;
    for (int t = 0; t <= T; ++t) s += part[t];
    free(part);
    return s;
}

/* Support restricted to the alive subgraph: common neighbours w of (a,b)
 * such that both edges (a,w) and (b,w) are alive.  Merge over full rows. */
static uint32_t alive_support(const int64_t* ptr, const int32_t* col, const int32_t* eid,
                              const uint8_t* alive, int32_t a, int32_t b) {
    int64_t i = ptr[a], i1 = ptr[a + 1], j = ptr[b], j1 = ptr[b + 1];
    uint32_t c = 0;
    int64_t na = i1 - i, nb = j1 - j;
    if (na > nb) { int64_t t; t = i; i = j; j = t; t = i1; i1 = j1; j1 = t; t = na; na = nb; nb = t; }
    if (nb >= 32 * na) {
        for (; i < i1; ++i) {
            int64_t p = lower_bound32(col, j, j1, col[i]);
            if (p < j1 && col[p] == col[i] && alive[eid[i]] && alive[eid[p]]) ++c;
        }
        return c;
    }
    while (i < i1 && j < j1) {
        if (col[i] < col[j]) ++i;
        else if (col[i] > col[j]) ++j;
        else { if (alive[eid[i]] && alive[eid[j]]) ++c; ++i; ++j; }
    }
    return c;
}

typedef struct { const int64_t* ptr; const int32_t* col; const int32_t* eid; const int32_t* cu; const int32_t* cv;
                 const uint8_t* alive; uint32_t* s; } rs_ctx;
static void rs_range(void* c, int64_t e0, int64_t e1, int t) {
    (void)t;
    rs_ctx* C = (rs_ctx*)c;
    for (int64_t e = e0; e < e1; ++e)
        C->s[e] = C->alive[e] ? alive_support(C->ptr, C->col, C->eid, C->alive, C->cu[e], C->cv[e]) : 0;
}

/* One Alg. 4 peel at threshold k, starting from `alive` (updated in place).
 * Each round recomputes s on the alive subgraph for every alive edge
 * (s = (R==2)·1 with R = E·A of the alive graph), then
 * removes x = {alive e : s(e) < k-2} as a batch.
 * removed_level (optional): set to `level_tag` for edges removed here.
 * trace (optional, cap trace_cap): |x| per round.
 * work (optional, 2 entries, accumulated): the k-truss byte model's terms
 * (SURVEY §8(d)): work[0] += Σ over rounds, over e = (a,b) in x with
 * s(e) > 0, of min(d(a), d(b)), d = alive degree at the round start;
 * work[1] += D, the support decrements: Σ over rounds of the drop of s on the
 * edges that stay (s at this round's recompute minus s at the next).
 * Returns #rounds with non-empty x. */
static int64_t peel_batch(int64_t n, int64_t m, const int32_t* cu, const int32_t* cv,
                          const int64_t* ptr, const int32_t* col, const int32_t* eid,
                          int32_t k, uint8_t* alive, uint32_t* s,
                          int32_t* removed_level, int32_t level_tag,
                          int64_t* trace, int64_t trace_cap, int64_t trace_base, int nthreads,
                          int64_t* work) {
    int64_t rounds = 0;
    uint32_t* prev = NULL;
    int64_t* d = NULL;
    if (work) {
        prev = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m > 0 ? m : 1));
        d = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    }
    int have_prev = 0;
    for (;;) {
        rs_ctx C = {ptr, col, eid, cu, cv, alive, s};
        parallel_for(m, nthreads, rs_range, &C);
        if (work && have_prev)
            for (int64_t e = 0; e < m; ++e)
                if (alive[e]) work[1] += (int64_t)prev[e] - (int64_t)s[e];
        int64_t nx = 0;
        if (work) {
            for (int64_t x = 0; x < n; ++x) d[x] = 0;
            for (int64_t e = 0; e < m; ++e)
                if (alive[e]) { d[cu[e]]++; d[cv[e]]++; }
        }
        /* x is decided for all edges before any is removed (batch) */
        for (int64_t e = 0; e < m; ++e)
            if (alive[e] && (int64_t)s[e] < (int64_t)k - 2) {
                if (work && s[e] > 0) work[0] += d[cu[e]] < d[cv[e]] ? d[cu[e]] : d[cv[e]];
                s[e] = 0xFFFFFFFFu;
                ++nx;
            }
        if (nx == 0) break;
        if (work) { memcpy(prev, s, sizeof(uint32_t) * (size_t)m); have_prev = 1; }
        for (int64_t e = 0; e < m; ++e)
            if (alive[e] && s[e] == 0xFFFFFFFFu) {
                alive[e] = 0;
                if (removed_level) removed_level[e] = level_tag;
            }
        if (trace && trace_base + rounds < trace_cap) trace[trace_base + rounds] = nx;
        ++rounds;
    }
    free(prev);
    free(d);
    return rounds;
}

/* ------------------------------------------------------------------ O-5 --
 * Maximal k-truss (reading A2), k >= 2.  alive_out: m (1 = kept).
 * trace: |x| per round (may be NULL).  work: see peel_batch (may be NULL).
 * Returns the number of rounds, or -1 for k < 2 (domain error). */
int64_t or_ktruss(int64_t n, int64_t m, const int32_t* cu, const int32_t* cv,
                  const int64_t* ptr, const int32_t* col, const int32_t* eid,
                  int32_t k, uint8_t* alive_out, int64_t* trace, int64_t trace_cap, int nthreads,
                  int64_t* work) {
    if (k < 2) return -1;
    for (int64_t e = 0; e < m; ++e) alive_out[e] = 1;
    uint32_t* s = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m > 0 ? m : 1));
    if (work) work[0] = work[1] = 0;
    int64_t r = peel_batch(n, m, cu, cv, ptr, col, eid, k, alive_out, s, NULL, 0, trace, trace_cap, 0, nthreads,
                           work);
    free(s);
    return r;
}

/* ------------------------------------------------------------------ O-6 --
 * Truss decomposition: run the k-truss with k = 3 on the full
 * graph, then pass the result to k+1, until empty.  tau(e) = k-1 for edges
 * removed at level k (so every edge has tau >= 2).  kmax = max tau, 0 when
 * m == 0 (reading A7).  work: see peel_batch, summed over the levels (may
 * be NULL).  Returns total rounds. */
int64_t or_truss_decomposition(int64_t n, int64_t m, const int32_t* cu, const int32_t* cv,
                               const int64_t* ptr, const int32_t* col, const int32_t* eid,
                               int32_t* tau, int32_t* kmax_out, int nthreads, int64_t* work) {
    uint8_t* alive = (uint8_t*)malloc((size_t)(m > 0 ? m : 1));
    uint32_t* s = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m > 0 ? m : 1));
    for (int64_t e = 0; e < m; ++e) { alive[e] = 1; tau[e] = 2; }
    int64_t left = m, rounds = 0;
    int32_t kmax = 0;
    if (work) work[0] = work[1] = 0;
    for (int32_t k = 3; left > 0; ++k) {
        rounds += peel_batch(n, m, cu, cv, ptr, col, eid, k, alive, s, tau, k - 1, NULL, 0, 0, nthreads, work);
        left = 0;
        for (int64_t e = 0; e < m; ++e) left += alive[e];
    }
    for (int64_t e = 0; e < m; ++e) if (tau[e] > kmax) kmax = tau[e];
    *kmax_out = (m > 0) ? kmax : 0;
    free(alive); free(s);
    return rounds;
}

/* ------------------------------------------------------------------ O-7 --
 * Tier-2 decomposition: remove one edge at a time, always
 * one of minimum current support (bin-sort buckets as in Batagelj-Zaversnik
 * k-core).  When e = (a,b) is removed with current support s, tau(e) = s + 2;
 * every live triangle (e, f, g) loses e, so f and g each lose one unit of
 * support, unless already at e's level (they will be removed at the same
 * level).  Sequential removal destroys each triangle exactly once.  Equal to
 * O-6 by uniqueness of the maximal k-truss (readings A2/A8).
 *
 * The live triangles through e are N_live(a) ∩ N_live(b), a plain sorted-list
 * intersection: two-pointer merge, or a galloping search of the shorter row
 * in the longer one when that is at least 32x longer (same set, fewer steps;
 * the same rule as O-3).  Storage details that change neither the removal order
 * nor the arithmetic: rows keep their live entries at the front (a row
 * holding more than twice its live count + 16 drops its dead entries in
 * place, keeping the order); an edge's support and bucket slot sit side by
 * side (slot -1 = removed); the common neighbours of e are listed first and
 * then applied in the same order (e's removal changes no other edge's state,
 * so listing first is the same as applying while merging).
 *
 * sup_init: O-3 supports (m).  consume != 0: col/eid are used as the row
 * storage and left scrambled (saves 8 B per stored entry at C4/C5); else they
 * are copied.  Returns m, or -1 on OOM / m > INT32_MAX. */
#ifndef O7_GALLOP
#define O7_GALLOP 32
#endif
typedef struct { uint32_t s; int32_t pos; } o7_edge;

int64_t or_truss_sequential(int64_t n, int64_t m, const int32_t* cu, const int32_t* cv,
                            const int64_t* ptr, int32_t* col_in, int32_t* eid_in,
                            const uint32_t* sup_init, int32_t* tau, int32_t* kmax_out, int consume) {
    if (m == 0) { *kmax_out = 0; return 0; }
    if (m > INT32_MAX) return -1;
    int32_t* col = col_in;
    int32_t* eid = eid_in;
    if (!consume) {
        col = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * m));
        eid = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * m));
        if (!col || !eid) { free(col); free(eid); return -1; }
        memcpy(col, col_in, sizeof(int32_t) * (size_t)(2 * m));
        memcpy(eid, eid_in, sizeof(int32_t) * (size_t)(2 * m));
    }
    o7_edge* E = (o7_edge*)malloc(sizeof(o7_edge) * (size_t)m);
    int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    int64_t* len = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));   /* stored entries */
    int64_t* live = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));  /* live entries */
    int64_t cap = 1024;
    int32_t* hits = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap * 2);          /* (f, g) pairs of e */
    uint32_t smax = 0;
    for (int64_t e = 0; e < m; ++e) if (sup_init[e] > smax) smax = sup_init[e];
    int64_t* bin = (int64_t*)calloc((size_t)smax + 2, sizeof(int64_t));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * ((size_t)smax + 1));
    if (!E || !ord || !len || !live || !hits || !bin || !fill) {
        free(E); free(ord); free(len); free(live); free(hits); free(bin); free(fill);
        if (!consume) { free(col); free(eid); }
        return -1;
    }
    for (int64_t x = 0; x < n; ++x) len[x] = live[x] = ptr[x + 1] - ptr[x];
    for (int64_t e = 0; e < m; ++e) bin[sup_init[e] + 1]++;
    for (uint32_t s = 0; s <= smax; ++s) bin[s + 1] += bin[s];
    for (uint32_t s = 0; s <= smax; ++s) fill[s] = bin[s];
    for (int64_t e = 0; e < m; ++e) {
        E[e].s = sup_init[e];
        E[e].pos = (int32_t)fill[sup_init[e]]++;
        ord[E[e].pos] = (int32_t)e;
    }
    free(fill);
    int32_t kmax = 2;
    /* bin[s] = first position of bucket s among not-yet-processed slots */
    for (int64_t i = 0; i < m; ++i) {
        int64_t e = ord[i];
        uint32_t se = E[e].s;
        tau[e] = (int32_t)se + 2;
        if (tau[e] > kmax) kmax = tau[e];
        /* common neighbours w of a and b: (a,w), (b,w) */
        int32_t a = cu[e], b = cv[e];
        int64_t p = ptr[a], p1 = ptr[a] + len[a], q = ptr[b], q1 = ptr[b] + len[b];
        if (p1 - p > q1 - q) {                     /* p walks the shorter row */
            int64_t t;
            t = p; p = q; q = t; t = p1; p1 = q1; q1 = t;
        }
        int gallop = (q1 - q) >= O7_GALLOP * (p1 - p);
        int64_t nh = 0;
        for (; p < p1 && q < q1; ++p) {
            if (gallop) {
                q = gallop32(col, q, q1, col[p]);
                if (q >= q1) break;
            } else {
                while (q < q1 && col[q] < col[p]) ++q;
                if (q >= q1) break;
            }
            if (col[q] != col[p]) continue;
            if (nh == cap) {
                cap *= 2;
                int32_t* nhits = (int32_t*)realloc(hits, sizeof(int32_t) * (size_t)cap * 2);
                if (!nhits) { nh = -1; break; }
                hits = nhits;
            }
            hits[2 * nh] = eid[p]; hits[2 * nh + 1] = eid[q];
            __builtin_prefetch(&E[eid[p]]); __builtin_prefetch(&E[eid[q]]);
            ++nh; ++q;
        }
        if (nh < 0) break;
        /* live triangles (both other edges alive) cost each of them one unit */
        for (int64_t j = 0; j < nh; ++j) {
            int64_t f = hits[2 * j], g = hits[2 * j + 1];
            if (E[f].pos < 0 || E[g].pos < 0) continue;
            int64_t fg[2] = {f, g};
            for (int t = 0; t < 2; ++t) {
                int64_t h = fg[t];
                if (E[h].s > se) {
                    /* move h to the front of its bucket, then shrink it by one */
                    uint32_t sh = E[h].s;
                    int64_t first = bin[sh];
                    if (first < i + 1) first = i + 1;
                    int64_t hw = ord[first];
                    if (hw != h) {
                        ord[E[h].pos] = (int32_t)hw; E[hw].pos = E[h].pos;
                        ord[first] = (int32_t)h; E[h].pos = (int32_t)first;
                    }
                    bin[sh] = first + 1;
                    E[h].s = sh - 1;
                }
            }
        }
        E[e].pos = -1;                             /* removed */
        /* buckets below the next slot are exhausted */
        if (bin[se] < i + 1) bin[se] = i + 1;
        /* drop dead entries from a row that is mostly dead */
        int32_t ab[2] = {a, b};
        for (int t = 0; t < 2; ++t) {
            int32_t x = ab[t];
            live[x]--;
            if (len[x] > 2 * live[x] + 16) {
                int64_t w = ptr[x];
                for (int64_t r = ptr[x]; r < ptr[x] + len[x]; ++r)
                    if (E[eid[r]].pos >= 0) { col[w] = col[r]; eid[w] = eid[r]; ++w; }
                len[x] = w - ptr[x];
            }
        }
    }
    int ok = 1;
    for (int64_t e = 0; e < m; ++e) if (E[e].pos >= 0) { ok = 0; break; }   /* OOM mid-run */
    *kmax_out = kmax;
    free(E); free(bin); free(ord); free(len); free(live); free(hits);
    if (!consume) { free(col); free(eid); }
    return ok ? m : -1;
}

/* ------------------------------------------------------------------ O-8 --
 * Tier-2 decomposition, parallel: Alg. 4 with its incremental update
 * written element-wise.  Levels k = 3, 4, ...;
 * within a level, rounds: x = {alive e : s(e) < k-2} (batch, reading A4);
 * every triangle alive at the round start with at least one edge in x loses
 * those edges, so each of its surviving edges loses one unit of support --
 * Alg. 4's R -= E_x-block update, counted once per triangle (reading A5: the
 * triangle is handled by its smallest-id edge in x); the edges whose support
 * falls below k-2 form the next round's x; x is removed with trussness k-1.
 * A level whose first x would be empty is skipped (no support changes, so
 * every k up to min s + 2 finds the same survivors).  Edges of x are handled
 * by independent threads (static chunks; support decrements are atomic, so
 * the result does not depend on the thread count or order).  The live
 * triangles of e = (a,b) are N_live(a) ∩ N_live(b) by the same sorted-list
 * intersection as O-3 / O-7; rows drop dead entries when the live edge count
 * has halved.  Equal to O-6 and O-7 (uniqueness of the maximal k-truss);
 * pinned against both.  sup_init: O-3 supports (m).  col/eid are used as row
 * storage and left scrambled.  Returns the number of rounds, -1 on OOM. */
typedef struct {
    const int64_t* ptr; const int64_t* len; const int32_t* col; const int32_t* eid;
    const int32_t* cu; const int32_t* cv; uint8_t* st; uint32_t* S; uint32_t thr;
    const int32_t* x; int32_t* next; int64_t* nnext;
} o8_round;

static void o8_enumerate(void* c, int64_t i0, int64_t i1, int t) {
    (void)t;
    o8_round* R = (o8_round*)c;
    for (int64_t i = i0; i < i1; ++i) {
        const int32_t e = R->x[i];
        const int32_t a = R->cu[e], b = R->cv[e];
        int64_t p = R->ptr[a], p1 = R->ptr[a] + R->len[a], q = R->ptr[b], q1 = R->ptr[b] + R->len[b];
        if (p1 - p > q1 - q) { int64_t s; s = p; p = q; q = s; s = p1; p1 = q1; q1 = s; }
        const int gallop = (q1 - q) >= 32 * (p1 - p);
        for (; p < p1 && q < q1; ++p) {
            if (gallop) {
                q = lower_bound32(R->col, q, q1, R->col[p]);
                if (q >= q1) break;
            } else {
                while (q < q1 && R->col[q] < R->col[p]) ++q;
                if (q >= q1) break;
            }
            if (R->col[q] != R->col[p]) continue;
            const int32_t f = R->eid[p], g = R->eid[q];
            ++q;
            const uint8_t sf = R->st[f], sg = R->st[g];          /* 0 removed, 1 alive, 2 in x */
            if (sf == 0 || sg == 0) continue;                     /* not a live triangle */
            if ((sf == 2 && f < e) || (sg == 2 && g < e)) continue;   /* a smaller x edge handles it */
            const int32_t fg[2] = {f, g};
            const uint8_t sfg[2] = {sf, sg};
            for (int k = 0; k < 2; ++k) {
                if (sfg[k] != 1) continue;                        /* x edges are not decremented */
                const uint32_t old = __atomic_fetch_sub(&R->S[fg[k]], 1u, __ATOMIC_RELAXED);
                if (old == R->thr) {                              /* crossing: next round's x */
                    const int64_t slot = __atomic_fetch_add(R->nnext, 1, __ATOMIC_RELAXED);
                    R->next[slot] = fg[k];
                }
            }
        }
    }
}

/* level-start scan of the alive list, in T static chunks: chunk t keeps its
 * alive edges (in place) and lists its x edges; counts per chunk */
typedef struct {
    int32_t* L; int64_t nL; const uint8_t* st; const uint32_t* S; uint32_t thr; int T;
    int32_t* xbuf; int64_t* kept; int64_t* nx; uint32_t* smin;
} o8_scan;
static void o8_scan_chunk(void* c, int64_t t0, int64_t t1, int unused) {
    (void)unused;
    o8_scan* Q = (o8_scan*)c;
    for (int64_t t = t0; t < t1; ++t) {
        const int64_t i0 = Q->nL * t / Q->T, i1 = Q->nL * (t + 1) / Q->T;
        int64_t w = i0, nx = 0;
        uint32_t smin = 0xFFFFFFFFu;
        for (int64_t i = i0; i < i1; ++i) {
            const int32_t e = Q->L[i];
            if (!Q->st[e]) continue;
            Q->L[w++] = e;
            if (Q->S[e] < Q->thr) Q->xbuf[i0 + nx++] = e;   /* within the chunk's own range */
            else if (Q->S[e] < smin) smin = Q->S[e];
        }
        Q->kept[t] = w - i0;
        Q->nx[t] = nx;
        Q->smin[t] = smin;
    }
}

typedef struct { const int64_t* ptr; int64_t* len; int32_t* col; int32_t* eid; const uint8_t* st; } o8_compact;
static void o8_compact_rows(void* c, int64_t v0, int64_t v1, int t) {
    (void)t;
    o8_compact* C = (o8_compact*)c;
    for (int64_t v = v0; v < v1; ++v) {
        int64_t w = C->ptr[v];
        for (int64_t r = C->ptr[v]; r < C->ptr[v] + C->len[v]; ++r)
            if (C->st[C->eid[r]]) { C->col[w] = C->col[r]; C->eid[w] = C->eid[r]; ++w; }
        C->len[v] = w - C->ptr[v];
    }
}

/* O-8 checkpoint (run-time bookkeeping only, no arithmetic): the state at a
 * level start -- supports, edge states, trussness so far, k, kmax, rounds,
 * live count.  The live list (alive edges in increasing id) and the rows
 * (the adjacency without dead entries) are rebuilt from the states on resume;
 * neither their order nor the compaction state changes any result. */
typedef struct { int64_t magic, n, m, k, kmax, rounds, alive; } o8_ckpt_hdr;
static const int64_t O8_MAGIC = 0x4f382d636b707431LL;

static int o8_save(const char* path, int64_t n, int64_t m, int32_t k, int32_t kmax, int64_t rounds, int64_t alive,
                   const uint32_t* S, const uint8_t* st, const int32_t* tau) {
    char tmp[4096];
    snprintf(tmp, sizeof tmp, "%s.part", path);
    FILE* f = fopen(tmp, "wb");
    if (!f) return -1;
    o8_ckpt_hdr h = {O8_MAGIC, n, m, k, kmax, rounds, alive};
    int ok = fwrite(&h, sizeof h, 1, f) == 1 && fwrite(S, 4, (size_t)m, f) == (size_t)m &&
             fwrite(st, 1, (size_t)m, f) == (size_t)m && fwrite(tau, 4, (size_t)m, f) == (size_t)m;
    ok = (fclose(f) == 0) && ok;
    if (!ok || rename(tmp, path) != 0) return -1;
    return 0;
}

static int o8_load(const char* path, int64_t n, int64_t m, int32_t* k, int32_t* kmax, int64_t* rounds, int64_t* alive,
                   uint32_t* S, uint8_t* st, int32_t* tau) {
    FILE* f = fopen(path, "rb");
    if (!f) return 1;                                          /* no checkpoint: start */
    o8_ckpt_hdr h;
    int ok = fread(&h, sizeof h, 1, f) == 1 && h.magic == O8_MAGIC && h.n == n && h.m == m &&
             fread(S, 4, (size_t)m, f) == (size_t)m && fread(st, 1, (size_t)m, f) == (size_t)m &&
             fread(tau, 4, (size_t)m, f) == (size_t)m;
    fclose(f);
    if (!ok) return -1;
    *k = (int32_t)h.k; *kmax = (int32_t)h.kmax; *rounds = h.rounds; *alive = h.alive;
    return 0;
}

static double o8_now(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

int64_t or_truss_parallel_ckpt(int64_t n, int64_t m, const int32_t* cu, const int32_t* cv, const int64_t* ptr,
                               int32_t* col, int32_t* eid, const uint32_t* sup_init, int32_t* tau, int32_t* kmax_out,
                               int nthreads, const char* ckpt, double budget_s);

int64_t or_truss_parallel(int64_t n, int64_t m, const int32_t* cu, const int32_t* cv, const int64_t* ptr,
                          int32_t* col, int32_t* eid, const uint32_t* sup_init, int32_t* tau, int32_t* kmax_out,
                          int nthreads) {
    return or_truss_parallel_ckpt(n, m, cu, cv, ptr, col, eid, sup_init, tau, kmax_out, nthreads, NULL, 0.0);
}

/* ckpt (may be NULL): resume from that file if it exists; with budget_s > 0,
 * after at least one level of this call and budget_s seconds, save the state
 * there at the next level start and return -2 (unfinished). */
int64_t or_truss_parallel_ckpt(int64_t n, int64_t m, const int32_t* cu, const int32_t* cv, const int64_t* ptr,
                               int32_t* col, int32_t* eid, const uint32_t* sup_init, int32_t* tau, int32_t* kmax_out,
                               int nthreads, const char* ckpt, double budget_s) {
    if (m == 0) { *kmax_out = 0; return 0; }
    if (m > INT32_MAX) return -1;
    const int T = n_threads(nthreads);
    uint32_t* S = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m);
    uint8_t* st = (uint8_t*)malloc((size_t)m);
    int32_t* L = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);      /* alive edges (compacted) */
    int32_t* x = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    int32_t* nx = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    int64_t* len = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t* kept = (int64_t*)malloc(sizeof(int64_t) * (size_t)T);
    int64_t* cnx = (int64_t*)malloc(sizeof(int64_t) * (size_t)T);
    uint32_t* cmin = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T);
    if (!S || !st || !L || !x || !nx || !len || !kept || !cnx || !cmin) {
        free(S); free(st); free(L); free(x); free(nx); free(len); free(kept); free(cnx); free(cmin);
        return -1;
    }
    for (int64_t e = 0; e < m; ++e) { S[e] = sup_init[e]; st[e] = 1; L[e] = (int32_t)e; tau[e] = 2; }
    for (int64_t v = 0; v < n; ++v) len[v] = ptr[v + 1] - ptr[v];
    int64_t nL = m, alive = m, compact_at = m, rounds = 0;
    int32_t kmax = 2, k0 = 3;
    if (ckpt) {
        const int r = o8_load(ckpt, n, m, &k0, &kmax, &rounds, &alive, S, st, tau);
        if (r < 0) {
            free(S); free(st); free(L); free(x); free(nx); free(len); free(kept); free(cnx); free(cmin);
            return -3;                                         /* unreadable checkpoint */
        }
        if (r == 0) {                                          /* resume: live list and rows from the states */
            nL = 0;
            for (int64_t e = 0; e < m; ++e)
                if (st[e]) L[nL++] = (int32_t)e;
            o8_compact C = {ptr, len, col, eid, st};
            parallel_for(n, T, o8_compact_rows, &C);
            compact_at = alive;
        }
    }
    const double t_start = o8_now();
    int levels_here = 0;
    for (int32_t k = k0; alive > 0; ++k) {
        if (ckpt && budget_s > 0 && levels_here > 0 && o8_now() - t_start > budget_s) {
            const int w = o8_save(ckpt, n, m, k, kmax, rounds, alive, S, st, tau);
            free(S); free(st); free(L); free(x); free(nx); free(len); free(kept); free(cnx); free(cmin);
            return w == 0 ? -2 : -4;                           /* unfinished (saved) / save failed */
        }
        ++levels_here;
        const uint32_t thr = (uint32_t)(k - 2);
        /* the level's first x; min s over the rest (empty-level skip); L keeps the alive edges */
        o8_scan Q = {L, nL, st, S, thr, T, nx, kept, cnx, cmin};
        parallel_for(T, T, o8_scan_chunk, &Q);
        int64_t w = 0, nxs = 0;
        uint32_t smin = 0xFFFFFFFFu;
        for (int t = 0; t < T; ++t) {
            const int64_t i0 = nL * t / T;
            memmove(L + w, L + i0, sizeof(int32_t) * (size_t)kept[t]);
            memcpy(x + nxs, nx + i0, sizeof(int32_t) * (size_t)cnx[t]);
            w += kept[t];
            nxs += cnx[t];
            if (cmin[t] < smin) smin = cmin[t];
        }
        nL = w;
        if (nxs == 0) {
            if (smin != 0xFFFFFFFFu && smin + 2 > (uint32_t)k) k = (int32_t)smin + 2;   /* loop's ++k: smin + 3 */
            continue;
        }
        while (nxs > 0) {
            for (int64_t i = 0; i < nxs; ++i) st[x[i]] = 2;
            int64_t nn = 0;
            o8_round R = {ptr, len, col, eid, cu, cv, st, S, thr, x, nx, &nn};
            parallel_for_dynamic(nxs, T, 64, o8_enumerate, &R);
            for (int64_t i = 0; i < nxs; ++i) { st[x[i]] = 0; tau[x[i]] = k - 1; }
            if (k - 1 > kmax) kmax = k - 1;
            alive -= nxs;
            ++rounds;
            int32_t* t = x; x = nx; nx = t;                        /* next round's x: the crossings */
            nxs = nn;
            if (alive > 0 && alive * 2 <= compact_at) {           /* rows drop their dead entries */
                o8_compact C = {ptr, len, col, eid, st};
                parallel_for(n, T, o8_compact_rows, &C);
                compact_at = alive;
            }
        }
    }
    *kmax_out = kmax;
    free(S); free(st); free(L); free(x); free(nx); free(len); free(kept); free(cnx); free(cmin);
    return rounds;
}
