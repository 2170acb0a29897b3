/*
 * gen.c — seeded synthetic edge-list generators (input harness only).
 *
 * This module is shared by the CPU oracle (oracle/) and the CUDA path
 * (paper_1708_06866_b200/) as the ONLY common piece: it produces raw directed
 * pairs (u[i], v[i]) and holds none of the method's arithmetic (no
 * canonicalisation, no degrees, no intersections).  Every draw is a pure
 * function of (seed, counter), so the output is identical for any thread
 * count and on any machine.
 *
 * Generators:
 *   - R-MAT / Kronecker (Graph500 style; §II "Data Sets" P:122-125
 *     names Graph500/Kronecker generators without fixing a construction).
 *   - Erdős–Rényi G(n, p) by an exact integer pair test.
 *   - King grid: the paper's own M×M image graphs, each pixel joined to its
 *     8 neighbours (§IV-C-1 "Benchmarking on Synthetic Graph Data",
 *     P:408-410, Table II).
 *
 * Output is deliberately "raw": R-MAT keeps self-loops and duplicates; ER
 * emits each edge once with a hashed orientation.  Normalisation
 * (self loops removed, reverse edges added) is the method's job.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

/* SplitMix64 finalizer (Steele, Lea, Flood 2014). */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Counter-based hash h(seed, a, b): stateless, 3 finalizer rounds. */
uint64_t gen_hash(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t x = mix64(seed + 0x9E3779B97F4A7C15ULL);
    x = mix64(x ^ (a + 0x632BE59BD9B4E019ULL));
    return mix64(x ^ (b + 0xD6E8FEB86659FD93ULL));
}

static int default_threads(int nthreads) {
    if (nthreads > 0) return nthreads;
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    if (c < 1) c = 1;
    if (c > 256) c = 256;
    return (int)c;
}

/* ---------------------------------------------------------------- perm --
 * Seeded bijection on [0, 2^s): 4 rounds of (odd multiply + add) mod 2^s and
 * an xor-shift-right, each a bijection on s-bit words.  Plays the role of the
 * Graph500 vertex-label shuffle so vertex ids carry no degree information. */
typedef struct { uint64_t mul[4], add[4], mask; int s, sh; } perm_key;

static void perm_init(perm_key* K, uint64_t seed, int s) {
    K->s = s;
    K->mask = (s >= 64) ? ~0ULL : ((1ULL << s) - 1ULL);
    K->sh = (s + 1) / 2;
    for (int r = 0; r < 4; ++r) {
        K->mul[r] = gen_hash(seed, 0x5045524DULL, 2 * r) | 1ULL;
        K->add[r] = gen_hash(seed, 0x5045524DULL, 2 * r + 1);
    }
}

static inline uint32_t perm_apply(const perm_key* K, uint32_t x) {
    uint64_t y = x & K->mask;
    for (int r = 0; r < 4; ++r) {
        y = (y * K->mul[r] + K->add[r]) & K->mask;
        if (K->s >= 2) y ^= (y >> K->sh);
    }
    return (uint32_t)y;
}

uint32_t gen_vertex_perm(uint64_t seed, int s, uint32_t x) {
    if (s <= 0) return 0;
    perm_key K;
    perm_init(&K, seed, s);
    return perm_apply(&K, x);
}

/* ---------------------------------------------------------------- R-MAT -- */
typedef struct {
    int s; uint64_t seed; int permute;
    uint64_t ta, tab, tabc;     /* integer quadrant thresholds on 53-bit draws */
    perm_key pk;
    int64_t i0, i1;
    int32_t* u; int32_t* v;
} rmat_job;

static void* rmat_worker(void* arg) {
    rmat_job* J = (rmat_job*)arg;
    const uint64_t x0 = mix64(J->seed + 0x9E3779B97F4A7C15ULL);
    for (int64_t i = J->i0; i < J->i1; ++i) {
        uint64_t xi = mix64(x0 ^ ((uint64_t)i + 0x632BE59BD9B4E019ULL));   /* gen_hash(seed,i,l) prefix */
        uint32_t uu = 0, vv = 0;
        for (int l = 0; l < J->s; ++l) {
            uint64_t r = mix64(xi ^ ((uint64_t)l + 0xD6E8FEB86659FD93ULL)) >> 11;   /* 53 bits */
            /* quadrant q = 0:a (0,0)  1:b (0,1)  2:c (1,0)  3:d (1,1)  (branch-free) */
            uint32_t q = (uint32_t)(r >= J->ta) + (uint32_t)(r >= J->tab) + (uint32_t)(r >= J->tabc);
            const int sh = J->s - 1 - l;
            uu |= (q >> 1) << sh;
            vv |= (q & 1u) << sh;
        }
        if (J->permute) {
            uu = perm_apply(&J->pk, uu);
            vv = perm_apply(&J->pk, vv);
        }
        J->u[i] = (int32_t)uu;
        J->v[i] = (int32_t)vv;
    }
    return NULL;
}

/* R-MAT with 2^s vertices and nnz = edge_factor * 2^s raw directed pairs.
 * Returns 0 on success, -1 on bad arguments.  u, v: caller-owned, nnz each. */
int gen_rmat(int s, int64_t nnz, double a, double b, double c, uint64_t seed,
             int permute, int32_t* u, int32_t* v, int nthreads) {
    if (s < 1 || s > 30 || nnz < 0 || a < 0 || b < 0 || c < 0 || a + b + c > 1.0) return -1;
    const double two53 = 9007199254740992.0;
    rmat_job proto;
    proto.s = s; proto.seed = seed; proto.permute = permute;
    proto.ta = (uint64_t)(a * two53);
    proto.tab = (uint64_t)((a + b) * two53);
    proto.tabc = (uint64_t)((a + b + c) * two53);
    proto.u = u; proto.v = v;
    perm_init(&proto.pk, seed ^ 0xA5A5A5A5DEADBEEFULL, s);
    int T = default_threads(nthreads);
    if (nnz < 4096) T = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * T);
    rmat_job* jobs = (rmat_job*)malloc(sizeof(rmat_job) * T);
    for (int t = 0; t < T; ++t) {
        jobs[t] = proto;
        jobs[t].i0 = nnz * t / T;
        jobs[t].i1 = nnz * (t + 1) / T;
        pthread_create(&th[t], NULL, rmat_worker, &jobs[t]);
    }
    for (int t = 0; t < T; ++t) pthread_join(th[t], NULL);
    free(th); free(jobs);
    return 0;
}

/* ------------------------------------------------------------------ ER --- */
typedef struct {
    int64_t n; uint64_t seed; uint64_t thr;
    int64_t r0, r1;            /* rows [r0, r1) */
    int64_t count;             /* pass 1 output */
    int64_t off;               /* pass 2 write offset */
    int32_t* u; int32_t* v;
} er_job;

static void* er_count(void* arg) {
    er_job* J = (er_job*)arg;
    int64_t cnt = 0;
    const uint64_t x0 = mix64(J->seed + 0x9E3779B97F4A7C15ULL);
    for (int64_t i = J->r0; i < J->r1; ++i) {
        const uint64_t xi = mix64(x0 ^ ((uint64_t)i + 0x632BE59BD9B4E019ULL));  /* == gen_hash prefix */
        for (int64_t j = i + 1; j < J->n; ++j)
            if (mix64(xi ^ ((uint64_t)j + 0xD6E8FEB86659FD93ULL)) < J->thr) ++cnt;
    }
    J->count = cnt;
    return NULL;
}

static void* er_fill(void* arg) {
    er_job* J = (er_job*)arg;
    int64_t k = J->off;
    const uint64_t x0 = mix64(J->seed + 0x9E3779B97F4A7C15ULL);
    for (int64_t i = J->r0; i < J->r1; ++i) {
        const uint64_t xi = mix64(x0 ^ ((uint64_t)i + 0x632BE59BD9B4E019ULL));
        for (int64_t j = i + 1; j < J->n; ++j) {
            uint64_t h = mix64(xi ^ ((uint64_t)j + 0xD6E8FEB86659FD93ULL));   /* gen_hash(seed,i,j) */
            if (h < J->thr) {
                /* orientation from the lowest bit of the same draw (the test uses the top bits) */
                if (h & 1ULL) {
                    J->u[k] = (int32_t)j; J->v[k] = (int32_t)i;
                } else {
                    J->u[k] = (int32_t)i; J->v[k] = (int32_t)j;
                }
                ++k;
            }
        }
    }
    return NULL;
}

/* Split rows so each thread gets ~equal pair counts (row i has n-1-i pairs). */
static void er_split(int64_t n, int T, er_job* jobs) {
    double total = (double)n * (double)(n - 1) / 2.0;
    int64_t r = 0;
    for (int t = 0; t < T; ++t) {
        jobs[t].r0 = r;
        double target = total * (double)(t + 1) / (double)T;
        if (t == T - 1) { r = n; }
        else {
            /* pairs in rows [0, r) = r*n - r(r+1)/2 ; advance until >= target */
            while (r < n && ((double)r * (double)n - (double)r * (double)(r + 1) / 2.0) < target) ++r;
        }
        jobs[t].r1 = r;
    }
}

/* Pass 1: number of edges of G(n, p) for this seed.  thr = floor(p * 2^64). */
int64_t gen_er_count(int64_t n, double p, uint64_t seed, int nthreads) {
    if (n < 0 || p < 0 || p >= 1.0) return -1;
    uint64_t thr = (uint64_t)(p * 18446744073709551616.0);
    int T = default_threads(nthreads);
    if (n < 512) T = 1;
    er_job* jobs = (er_job*)calloc(T, sizeof(er_job));
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * T);
    er_split(n, T, jobs);
    for (int t = 0; t < T; ++t) {
        jobs[t].n = n; jobs[t].seed = seed; jobs[t].thr = thr;
        pthread_create(&th[t], NULL, er_count, &jobs[t]);
    }
    int64_t tot = 0;
    for (int t = 0; t < T; ++t) { pthread_join(th[t], NULL); tot += jobs[t].count; }
    free(jobs); free(th);
    return tot;
}

/* Pass 2: fill u, v (capacity cap, must be >= gen_er_count result).
 * Edges come out in (min, max) lexicographic order with hashed orientation.
 * Returns the number written or -1. */
int64_t gen_er_fill(int64_t n, double p, uint64_t seed, int32_t* u, int32_t* v,
                    int64_t cap, int nthreads) {
    if (n < 0 || p < 0 || p >= 1.0) return -1;
    uint64_t thr = (uint64_t)(p * 18446744073709551616.0);
    int T = default_threads(nthreads);
    if (n < 512) T = 1;
    er_job* jobs = (er_job*)calloc(T, sizeof(er_job));
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * T);
    er_split(n, T, jobs);
    for (int t = 0; t < T; ++t) {
        jobs[t].n = n; jobs[t].seed = seed; jobs[t].thr = thr;
        pthread_create(&th[t], NULL, er_count, &jobs[t]);
    }
    int64_t off = 0;
    for (int t = 0; t < T; ++t) { pthread_join(th[t], NULL); jobs[t].off = off; off += jobs[t].count; }
    if (off > cap) { free(jobs); free(th); return -1; }
    for (int t = 0; t < T; ++t) {
        jobs[t].u = u; jobs[t].v = v;
        pthread_create(&th[t], NULL, er_fill, &jobs[t]);
    }
    for (int t = 0; t < T; ++t) pthread_join(th[t], NULL);
    free(jobs); free(th);
    return off;
}

/* ------------------------------------------------------------ king grid --
 * M×M pixels, pixel (r, c) -> id r*M + c, joined to its 8 neighbours
 * (P:408-410).  Emits each undirected edge once (right, down, down-right,
 * down-left), 2(M-1)(2M-1) pairs.  Returns the count written. */
int64_t gen_king_grid(int64_t M, int32_t* u, int32_t* v) {
    int64_t k = 0;
    for (int64_t r = 0; r < M; ++r)
        for (int64_t c = 0; c < M; ++c) {
            int64_t x = r * M + c;
            if (c + 1 < M) { u[k] = (int32_t)x; v[k] = (int32_t)(x + 1); ++k; }
            if (r + 1 < M) { u[k] = (int32_t)x; v[k] = (int32_t)(x + M); ++k; }
            if (r + 1 < M && c + 1 < M) { u[k] = (int32_t)x; v[k] = (int32_t)(x + M + 1); ++k; }
            if (r + 1 < M && c >= 1) { u[k] = (int32_t)x; v[k] = (int32_t)(x + M - 1); ++k; }
        }
    return k;
}
