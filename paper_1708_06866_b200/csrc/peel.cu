// peel.cu — incremental k-truss peeler and truss decomposition (SURVEY
// §8(a) rows a8, a9).
//
// Method: P:247 [k-Truss] "each edge is contained in at least (k-2)
// triangles in the same subgraph"; Alg. 4 removes, per round,
// the whole vector x = find(s < k-2) and updates R = EA by subtracting the
// removed edges' contribution instead of recomputing it.  The
// element-wise meaning of that update: every triangle alive at the start of
// the round that loses at least one edge costs each of its surviving edges
// exactly one unit of support.  On the GPU:
//
//   frontier X (edges with s < k-2, alive)                   -- Alg. 4 "x"
//   one warp per e in X: enumerate the live triangles through e by searching
//     the shorter endpoint row in the longer one (symmetric CSR, rank space);
//     a triangle with several edges in X is handled only by its smallest-id
//     edge in X (reading A5), which decrements each survivor once
//     (atomicSub); a survivor crossing from k-2 to k-3 joins the next
//     frontier (threshold crossing: no full rescan per round)
//   alive -= X
//
// until X is empty (fixed point).  Decomposition: k = 3, 4, ...
// continue from the previous k's survivors; edges removed at level k get
// trussness k-1.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_profiler_api.h>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstring>

#include "gc_internal.cuh"

namespace gcx {

namespace {

__global__ void k_sym_fill(const int32_t* __restrict__ in_src, const int32_t* __restrict__ in_dst,
                           const int32_t* __restrict__ in_pos, const int32_t* __restrict__ dag_src,
                           const int32_t* __restrict__ dag_col, const int64_t* __restrict__ dag_ptr,
                           const int64_t* __restrict__ in_ptr, int64_t m, int32_t* __restrict__ col,
                           int32_t* __restrict__ eid) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        // lower part of row x = in_dst[i]: slot dag_ptr[x] + i
        int x = in_dst[i];
        int64_t s = dag_ptr[x] + i;
        col[s] = in_src[i];
        eid[s] = in_pos[i];
        // upper part of row y = dag_src[i] (DAG position i): slot in_ptr[y+1] + i
        int y = dag_src[i];
        int64_t t = in_ptr[y + 1] + i;
        col[t] = dag_col[i];
        eid[t] = (int32_t)i;
    }
}

__global__ void k_sym_ptr(const int64_t* __restrict__ dag_ptr, const int64_t* __restrict__ in_ptr, int64_t n,
                          int64_t* __restrict__ sym_ptr) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n; x += (int64_t)gridDim.x * blockDim.x)
        sym_ptr[x] = dag_ptr[x] + in_ptr[x];
}

__global__ void k_fill_u8(uint8_t* __restrict__ a, int64_t m, uint8_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) a[i] = v;
}

__global__ void k_fill_i32(int32_t* __restrict__ a, int64_t m, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) a[i] = v;
}

// ------------------------------------------------ dead-entry compaction --
// As edges die, the symmetric rows fill with dead entries that every later
// triangle search would still walk.  When the live edge count has halved
// since the last compaction, each row's live entries are moved (stably, so
// rows stay sorted) to the front of its own segment and live_len[x] records
// the new length; the list of live edges is rebuilt for the level scans.
__global__ void k_live_len_init(const int64_t* __restrict__ sym_ptr, int64_t n, int32_t* __restrict__ live_len) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
        live_len[x] = (int32_t)(sym_ptr[x + 1] - sym_ptr[x]);
}

constexpr int kLongRow = 2048;   // rows longer than this are compacted by a whole block

__global__ void k_long_rows(const int64_t* __restrict__ sym_ptr, int64_t n, int32_t* __restrict__ list,
                            int* __restrict__ count) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
        if (sym_ptr[x + 1] - sym_ptr[x] > kLongRow) list[atomicAdd(count, 1)] = (int32_t)x;
}

// one warp per row of at most kLongRow live entries; in place: each chunk of
// 32 is read by the warp before any of it is written (writes never pass reads)
__global__ void k_row_compact_warp(const int64_t* __restrict__ sym_ptr, int32_t* __restrict__ live_len,
                                   int32_t* __restrict__ col, int32_t* __restrict__ eid,
                                   const uint8_t* __restrict__ alive, int64_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t x = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; x < n; x += nw) {
        const int L = live_len[x];
        if (L > kLongRow || L == 0) continue;
        const int64_t base = sym_ptr[x];
        int out = 0;
        for (int i0 = 0; i0 < L; i0 += 32) {
            const int i = i0 + lane;
            int cv = 0, ev = 0;
            bool keep = false;
            if (i < L) {
                cv = col[base + i];
                ev = eid[base + i];
                keep = alive[ev] != 0;
            }
            const unsigned b = __ballot_sync(0xffffffffu, keep);
            __syncwarp();
            if (keep) {
                const int o = out + __popc(b & ((1u << lane) - 1));
                col[base + o] = cv;
                eid[base + o] = ev;
            }
            out += __popc(b);
        }
        if (lane == 0) live_len[x] = out;
    }
}

// one block per long row (list built once with the symmetric CSR)
__global__ void __launch_bounds__(256) k_row_compact_block(const int32_t* __restrict__ rows, int nrows,
                                                            const int64_t* __restrict__ sym_ptr,
                                                            int32_t* __restrict__ live_len, int32_t* __restrict__ col,
                                                            int32_t* __restrict__ eid,
                                                            const uint8_t* __restrict__ alive) {
    __shared__ int wsum[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int x = rows[r];
        const int L = live_len[x];
        if (L <= kLongRow) continue;            // uniform per block
        const int64_t base = sym_ptr[x];
        int out = 0;
        for (int i0 = 0; i0 < L; i0 += 256) {
            const int i = i0 + threadIdx.x;
            int cv = 0, ev = 0;
            bool keep = false;
            if (i < L) {
                cv = col[base + i];
                ev = eid[base + i];
                keep = alive[ev] != 0;
            }
            const unsigned b = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) wsum[warp] = __popc(b);
            __syncthreads();
            int before = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                before += w < warp ? wsum[w] : 0;
                tot += wsum[w];
            }
            if (keep) {
                const int o = out + before + __popc(b & ((1u << lane) - 1));
                col[base + o] = cv;
                eid[base + o] = ev;
            }
            out += tot;
            __syncthreads();                    // wsum reuse; this chunk's writes precede the next chunk's reads
        }
        if (threadIdx.x == 0) live_len[x] = out;
    }
}

__global__ void k_alive_list(const uint8_t* __restrict__ alive, int64_t m, int32_t* __restrict__ list,
                             int* __restrict__ count) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const bool in = alive[e] != 0;
        const unsigned ballot = __ballot_sync(__activemask(), in);
        if (in) {
            const int lane = threadIdx.x & 31, leader = __ffs(ballot) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(count, __popc(ballot));
            base = __shfl_sync(ballot, base, leader);
            list[base + __popc(ballot & ((1u << lane) - 1))] = (int32_t)e;
        }
    }
}

// Edge state, one byte per edge (the alive array): 0 removed, 1 alive, and
// st_front(r) = 2 + (r & 1) alive and in the frontier X of round r.  Crossings
// during round r are stamped st_front(r + 1), which no edge of round r's X
// carries, and X turns 0 when the round finishes, so two values suffice and a
// triangle visit reads one byte per other edge for both "alive" and "in X"
// (5x less state than a separate int32 round stamp: the dense cores' states
// stay in L2).
__host__ __device__ __forceinline__ uint8_t st_front(int32_t round) { return (uint8_t)(2 + (round & 1)); }

// X = {alive e : S(e) < thr}, over the live-edge list (list == nullptr: all e < m)
// An edge below the threshold with S(e) = 0 lies in no live triangle, so it
// is removed on the spot (nothing to destroy, nobody sees it in this round);
// the others go to the frontier list for the peel kernel.
// Level scan: every alive edge of [0, len) (or of list) with S = 0 leaves on
// the spot (no triangle, no decrement); the others with S < thr form the
// round's frontier X.  Two passes over each warp's contiguous slice: the
// first applies the removals, counts X and keeps each 32-edge step's ballot
// in shared memory, the block takes its whole range with ONE global atomic,
// the second writes X in slice order at the ballots' offsets (no re-read of
// S or alive) -- no per-tile barrier or atomic (one atomic per 256-edge tile,
// on a single counter, made the C4 k = 4 scan 2.9 ms for 1.3 GB of reads).
constexpr int kScanSteps = 512;    // ballots kept per warp (slices up to 16,384 edges)
__global__ void __launch_bounds__(256) k_frontier_scan(const uint32_t* __restrict__ S, uint8_t* __restrict__ alive,
                                const int32_t* __restrict__ list, int64_t len, uint32_t thr,
                                int32_t round, int32_t* __restrict__ front,
                                int* __restrict__ count, int32_t* __restrict__ tau, int32_t level,
                                unsigned long long* __restrict__ zero_removed, uint32_t* __restrict__ min_rest,
                                int32_t* __restrict__ zlist, int* __restrict__ zcount) {
    __shared__ int woff[8];
    __shared__ int bbase;
    __shared__ unsigned bal[8][kScanSteps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // this block's range, cut into 8 warp slices (multiples of 32)
    const int64_t per_block = ((len + gridDim.x - 1) / gridDim.x + 255) & ~(int64_t)255;
    const int64_t b0 = (int64_t)blockIdx.x * per_block;
    const int64_t per_warp = per_block / 8;
    const int64_t w0 = min(len, b0 + warp * per_warp), w1 = min(len, w0 + per_warp);
    unsigned zeros = 0;
    uint32_t rest = 0xFFFFFFFFu;   // min S over the alive edges left out of the frontier
    int mine = 0;
    const bool keep = (w1 - w0 + 31) / 32 <= kScanSteps;
    for (int64_t i0 = w0; i0 < w1; i0 += 32) {          // pass 1: removals, count X
        const int64_t i = i0 + lane;
        bool in = false;
        if (i < w1) {
            const int64_t e = list ? (int64_t)list[i] : i;
            if (alive[e]) {
                const uint32_t se = S[e];
                if (se == 0 && thr > 0) {
                    alive[e] = 0;
                    if (tau) tau[e] = level;
                    if (zlist) zlist[atomicAdd(zcount, 1)] = (int32_t)e;   // work stats only
                    ++zeros;
                } else {
                    in = se < thr;
                    if (!in) rest = min(rest, se);
                }
            }
        }
        const unsigned b = __ballot_sync(0xffffffffu, in);
        if (keep && lane == 0) bal[warp][(i0 - w0) >> 5] = b;
        mine += __popc(b);
    }
    if (lane == 0) woff[warp] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < 8; ++w) {
            const int c = woff[w];
            woff[w] = tot;
            tot += c;
        }
        bbase = tot ? atomicAdd(count, tot) : 0;
    }
    __syncthreads();
    if (mine && keep) {
        int off = bbase + woff[warp];
        for (int64_t i0 = w0; i0 < w1; i0 += 32) {      // pass 2: X in slice order, from the ballots
            const unsigned b = bal[warp][(i0 - w0) >> 5];
            if (!b) continue;
            if ((b >> lane) & 1u) {
                const int64_t i = i0 + lane;
                const int64_t e = list ? (int64_t)list[i] : i;
                alive[e] = st_front(round);
                front[off + __popc(b & ((1u << lane) - 1))] = (int32_t)e;
            }
            off += __popc(b);
        }
    } else if (mine) {
        int off = bbase + woff[warp];
        for (int64_t i0 = w0; i0 < w1; i0 += 32) {      // pass 2: X in slice order
            const int64_t i = i0 + lane;
            bool in = false;
            int64_t e = -1;
            if (i < w1) {
                e = list ? (int64_t)list[i] : i;
                in = alive[e] && S[e] < thr;             // zero-support edges are gone (alive = 0) by now
            }
            const unsigned ballot = __ballot_sync(0xffffffffu, in);
            if (in) {
                alive[e] = st_front(round);
                front[off + __popc(ballot & ((1u << lane) - 1))] = (int32_t)e;
            }
            off += __popc(ballot);
        }
    }
    zeros = __reduce_add_sync(0xffffffffu, zeros);
    if (lane == 0 && zeros) atomicAdd(zero_removed, (unsigned long long)zeros);
    rest = __reduce_min_sync(0xffffffffu, rest);
    if (lane == 0 && rest != 0xFFFFFFFFu) atomicMin(min_rest, rest);
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* __restrict__ a, int64_t lo, int64_t hi, int32_t x) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Round semantics (reading A5): a triangle alive at the round start with at
// least one edge in X is handled only by its smallest-id edge in X, which
// decrements each surviving edge once.  The two policies differ in how X is
// represented and which survivors a rank may decrement.
struct PolicySingle {       // one rank: X = {st == st_front(round)}; crossings append to the next list
    uint8_t* st;            // the alive array (edge state, see st_front)
    uint32_t* S;
    uint32_t thr;
    int32_t round;
    int32_t* next;
    int* next_count;
    __device__ __forceinline__ uint32_t live(int e) const { return S[e]; }   // exact at round start
    __device__ __forceinline__ bool in_x(int f) const { return st[f] == st_front(round); }
    __device__ __forceinline__ void dec(int f) const {
        if (atomicSub(S + f, 1u) == thr) {
            st[f] = st_front(round + 1);
            next[atomicAdd(next_count, 1)] = f;   // (warp-aggregating this append cost the decomposition 1 %)
        }
    }
    // both survivors of a triangle: the two atomics in flight together (each
    // returns the old support for the crossing test, so one after the other
    // the second waited out the first's round trip)
    __device__ __forceinline__ void dec2(int f, int g) const {
        const uint32_t of = atomicSub(S + f, 1u), og = atomicSub(S + g, 1u);
        if (of == thr) {
            st[f] = st_front(round + 1);
            next[atomicAdd(next_count, 1)] = f;
        }
        if (og == thr) {
            st[g] = st_front(round + 1);
            next[atomicAdd(next_count, 1)] = g;
        }
    }
};

// P owners of contiguous, word-aligned DAG-position slices (§8(e); the
// enumeration partitioned by owner, §8(f) #1 "v2"): X travels as a bitmap,
// each X edge is enumerated by its owner only (its S is exact there: early
// exit), and a decrement lands on the survivor's owner copy -- directly for
// loopback virtual ranks (one device), through a list exchanged after the
// chunk for another NCCL rank.
struct PolicyPart {
    const uint32_t* xbits;
    uint32_t* S;            // owner copies: owner o's at S + o * stride (loopback: stride m; NCCL: own copy, stride 0)
    int64_t stride;
    int64_t span;           // edges per owner slice (32 W)
    int me;                 // NCCL: this rank; -1: loopback (every owner on this device)
    uint32_t thr;
    uint32_t* nbits;        // next X: crossings set their bit (owner's slice)
    int32_t* out;           // NCCL: decrements of other ranks' edges
    unsigned long long* out_n;
    int64_t out_cap;
    __device__ __forceinline__ int owner(int64_t e) const { return (int)(e / span); }
    __device__ __forceinline__ uint32_t live(int e) const { return S[(int64_t)owner(e) * stride + e]; }
    __device__ __forceinline__ bool in_x(int f) const { return (xbits[f >> 5] >> (f & 31)) & 1u; }
    __device__ __forceinline__ void dec2(int f, int g) const {
        dec(f);
        dec(g);
    }
    __device__ __forceinline__ void dec(int f) const {
        const int o = owner(f);
        if (me < 0 || o == me) {
            if (atomicSub(S + (int64_t)o * stride + f, 1u) == thr) atomicOr(nbits + (f >> 5), 1u << (f & 31));
        } else {
            const unsigned long long i = atomicAdd(out_n, 1ULL);
            if ((int64_t)i < out_cap) out[i] = f;
        }
    }
};

template <class Pol>
__device__ __forceinline__ void destroy(const Pol& pol, int e, int f, int g) {
    const bool fx = pol.in_x(f), gx = pol.in_x(g);
    if ((fx && f < e) || (gx && g < e)) return;   // a smaller X-edge owns this triangle
    if (!fx && !gx) {
        pol.dec2(f, g);
    } else {
        if (!fx) pol.dec(f);
        if (!gx) pol.dec(g);
    }
}

struct PeelArgs {
    const int32_t* front;
    int nfront;
    const int* nfront_dev;  // non-null: the frontier size is read on the device (rounds enqueued ahead)
    const int32_t* dag_src;
    const int32_t* dag_col;
    const int64_t* sym_ptr;
    const int32_t* live_len;
    const int32_t* sym_col;
    const int32_t* sym_eid;
    const uint8_t* alive;
};

// Destroy the live triangles of each frontier edge e = (a, b): walk the
// shorter endpoint row -- from its end: the highest-ranked (highest-degree)
// third vertices close most triangles -- and binary-search each live entry
// in the longer one (rows sorted by rank; dead entries compacted away now
// and then).  Stop once S(e) live triangles are found (S exact for the
// edges a rank enumerates).  A warp takes G frontier edges at a time (G = 1 for small
// frontiers, up to 32 for big ones): lanes whose shorter row has at most
// kSerialRow entries walk it alone (uniform-degree graphs: every lane busy),
// the other edges are walked by the whole warp one after another.  Measured
// alternatives: 32-ary window narrowing of the longer row and
// splitting long rows into work items over many warps were slower.
constexpr int kSerialRow = 8;
#ifndef GC_GRP_MINB
#define GC_GRP_MINB 4    // ... of k_peel_grouped (48 KB of shared memory per block)
#endif
#ifndef GC_PEEL_REVERSE
#define GC_PEEL_REVERSE 1   // walk the shorter row from its end, highest ranks first (C4 k = 4 / 6 peel 39.3 -> 28.4 / 96.4 -> 61.6 ms,
                            // decomposition 1.59 -> 1.49 s; C5 decomposition 19.5 -> 18.7 s); 0: from its start
#endif
#ifndef GC_PEEL_FIRST32
#define GC_PEEL_FIRST32 1   // the walk's first step searches 32 entries, later ones 64 (C4 k = 4 / 6 peel -5 % / -6 %,
                            // C4 decomposition +1 %, C5 decomposition -1 %); 0: 64 from the start
#endif
#ifndef GC_PEEL_GMAX
#define GC_PEEL_GMAX 8   // frontier edges per warp at most (8: K13 kernel 226 -> 78 ms, C4 +0.7 %)
#endif


// Branch-free lower bounds of two targets in one sorted range, in lockstep:
// the halving sequence does not depend on the targets, so the two searches'
// loads are independent and in flight together (the peel's searches are
// latency-bound: C4 / C5 decomposition kernels -15 % / -12 %; a generic
// N-target version with register arrays needed more registers and was slower
// at 2, 3 and 4 targets).  r = smallest i in [lo, hi) with a[i] >= x, hi if none.
__device__ __forceinline__ void lower_bound_x2(const int32_t* __restrict__ a, int64_t lo, int64_t hi, int32_t x0,
                                               int32_t x1, int64_t& r0, int64_t& r1) {
    int64_t n = hi - lo;
    if (n <= 0) {
        r0 = r1 = lo;
        return;
    }
    int64_t p0 = lo, p1 = lo;
    while (n > 1) {
        const int64_t half = n >> 1;
        const int32_t v0 = __ldg(a + p0 + half), v1 = __ldg(a + p1 + half);
        p0 = v0 < x0 ? p0 + half : p0;
        p1 = v1 < x1 ? p1 + half : p1;
        n -= half;
    }
    r0 = p0 + (__ldg(a + p0) < x0);
    r1 = p1 + (__ldg(a + p1) < x1);
}

#ifndef GC_PEEL_PF
#define GC_PEEL_PF 0            // TMA bulk L2 prefetch (cp.async.bulk.prefetch.L2) of the next warp-walked edge's rows
#endif
#ifndef GC_PEEL_PF_MAX
#define GC_PEEL_PF_MAX 2048     // ... the searched (longer) row only up to this many entries
#endif
#if GC_PEEL_PF
// a[lo, hi) into L2 through the TMA unit (16-byte aligned superset; warp-uniform arguments)
__device__ __forceinline__ void row_pf(const int32_t* __restrict__ a, int64_t lo, int64_t hi) {
    const uintptr_t x = reinterpret_cast<uintptr_t>(a + lo) & ~(uintptr_t)15;
    const uintptr_t z = (reinterpret_cast<uintptr_t>(a + hi) + 15) & ~(uintptr_t)15;
    if (hi > lo) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x), "r"((uint32_t)(z - x)) : "memory");
}
#endif

template <class Pol>
__device__ __forceinline__ void peel_one_warp(const PeelArgs& A, const Pol& pol, int e, uint32_t live, int64_t a0,
                                              int64_t a1, int64_t b0, int64_t b1, int lane) {
    uint32_t found = 0;
    // two 32-entry chunks of the shorter row per step, their searches interleaved
#if GC_PEEL_REVERSE
    // from the row's end: high-rank (high-degree) third vertices close most
    // triangles, so an edge with few live triangles stops sooner
#if GC_PEEL_FIRST32
    // the first step takes only the top 32 entries: an edge with one or two
    // live triangles usually finds them there
    for (int64_t top = a1, step = 32; top > a0 && found < live; top -= step, step = 64) {
        const int64_t i0 = top - 64 + lane, i1 = top - 32 + lane;
        const bool in0 = step == 64 && i0 >= a0, in1 = i1 >= a0;
#else
    for (int64_t top = a1; top > a0 && found < live; top -= 64) {
        const int64_t i0 = top - 64 + lane, i1 = top - 32 + lane;
        const bool in0 = i0 >= a0, in1 = i1 >= a0;
#endif
#else
    for (int64_t base = a0; base < a1 && found < live; base += 64) {
        const int64_t i0 = base + lane, i1 = base + 32 + lane;
        const bool in0 = i0 < a1, in1 = i1 < a1;
#endif
        int f0 = -1, f1 = -1;
        int32_t w0 = INT32_MAX, w1 = INT32_MAX;
        if (in0) {
            f0 = __ldg(A.sym_eid + i0);
            w0 = __ldg(A.sym_col + i0);
        }
        if (in1) {
            f1 = __ldg(A.sym_eid + i1);
            w1 = __ldg(A.sym_col + i1);
        }
        const bool want0 = in0 && f0 != e && A.alive[f0];
        const bool want1 = in1 && f1 != e && A.alive[f1];
        bool tri0 = false, tri1 = false;
        int g0 = -1, g1 = -1;
        if (want0 || want1) {
            int64_t j0, j1;
            lower_bound_x2(A.sym_col, b0, b1, w0, w1, j0, j1);
            if (want0 && j0 < b1 && __ldg(A.sym_col + j0) == w0) {
                g0 = __ldg(A.sym_eid + j0);
                tri0 = A.alive[g0] != 0;
            }
            if (want1 && j1 < b1 && __ldg(A.sym_col + j1) == w1) {
                g1 = __ldg(A.sym_eid + j1);
                tri1 = A.alive[g1] != 0;
            }
        }
        found += __popc(__ballot_sync(0xffffffffu, tri0)) + __popc(__ballot_sync(0xffffffffu, tri1));
        if (tri0) destroy(pol, e, f0, g0);
        if (tri1) destroy(pol, e, f1, g1);
    }
}

// MINB: the register budget.  MINB = 8 (32 registers, the SM's 64 warps) is
// the build that runs: the searches are latency-bound, and with two of them
// in flight per lane it wins at every frontier size (C4 / C5 decomposition
// kernels 1.50 -> 1.40 s / 19.4 -> 17.4 s, C4 ktruss(6) peel 119 -> 99 ms
// against MINB = 1 for frontiers of 2^20 edges and more).  MINB = 1 stays
// reachable through GC_PEEL_BIG for A/B runs.
template <class Pol, int MINB>
__global__ void __launch_bounds__(256, MINB) k_peel(PeelArgs A, Pol pol) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nfront = A.nfront_dev ? *A.nfront_dev : A.nfront;
    if (nfront > 0 && 2 * (int64_t)nfront <= warps) {
        // Few frontier edges (the late rounds of the dense cores: a handful of
        // edges with long rows): each edge's shorter row is cut into wpe
        // 32-aligned slices, one per warp, so the whole grid works on them
        // instead of one warp per edge.  No early exit (S(e) counts the edge's
        // triangles across all slices); each triangle is still met once, in
        // the slice holding its entry of the shorter row.
        const int64_t wpe = warps / nfront;
        const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
        const int64_t ei = wid / wpe, slice = wid % wpe;
        if (ei >= nfront) return;
        const int e = A.front[ei];
        const uint32_t live = pol.live(e);
        if (live == 0) return;
        const int a = A.dag_src[e], b = A.dag_col[e];
        int64_t a0 = A.sym_ptr[a], a1 = a0 + A.live_len[a], b0 = A.sym_ptr[b], b1 = b0 + A.live_len[b];
        if (a1 - a0 > b1 - b0) {
            int64_t t0 = a0, t1 = a1;
            a0 = b0; a1 = b1; b0 = t0; b1 = t1;
        }
        const int64_t chunks = (a1 - a0 + 31) / 32;
        const int64_t c0 = chunks * slice / wpe, c1 = chunks * (slice + 1) / wpe;
        if (c1 > c0)
            peel_one_warp<Pol>(A, pol, e, 0xFFFFFFFFu, a0 + 32 * c0, min(a1, a0 + 32 * c1), b0, b1, lane);
        return;
    }
    const int G = (int)max((int64_t)1, min((int64_t)GC_PEEL_GMAX, nfront / warps));     // edges per warp
    for (int64_t base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * G; base < nfront;
         base += warps * G) {
        int e = -1;
        uint32_t live = 0;
        int64_t a0 = 0, a1 = 0, b0 = 0, b1 = 0;
        if (lane < G && base + lane < nfront) {
            e = A.front[base + lane];
            live = pol.live(e);
            if (live) {
                const int a = A.dag_src[e], b = A.dag_col[e];
                a0 = A.sym_ptr[a]; a1 = a0 + A.live_len[a]; b0 = A.sym_ptr[b]; b1 = b0 + A.live_len[b];
                if (a1 - a0 > b1 - b0) {
                    int64_t t0 = a0, t1 = a1;
                    a0 = b0; a1 = b1; b0 = t0; b1 = t1;
                }
            }
        }
        const bool serial = live && G > 1 && a1 - a0 <= kSerialRow;
        if (serial) {                                   // this lane alone
            uint32_t found = 0;
#if GC_PEEL_REVERSE
            int64_t hi = b1;
            for (int64_t i = a1 - 1; i >= a0 && found < live; --i) {
                const int f = __ldg(A.sym_eid + i);
                if (f == e || !A.alive[f]) continue;
                const int32_t w = __ldg(A.sym_col + i);
                const int64_t j = lower_bound_i32(A.sym_col, b0, hi, w);   // targets descend along the row
                if (j < hi && __ldg(A.sym_col + j) == w) {
                    const int g = __ldg(A.sym_eid + j);
                    if (A.alive[g]) {
                        ++found;
                        destroy(pol, e, f, g);
                    }
                }
                hi = j;
            }
#else
            int64_t lo = b0;
            for (int64_t i = a0; i < a1 && found < live; ++i) {
                const int f = __ldg(A.sym_eid + i);
                if (f == e || !A.alive[f]) continue;
                const int32_t w = __ldg(A.sym_col + i);
                lo = lower_bound_i32(A.sym_col, lo, b1, w);   // targets ascend along the row
                if (lo < b1 && __ldg(A.sym_col + lo) == w) {
                    const int g = __ldg(A.sym_eid + lo);
                    if (A.alive[g]) {
                        ++found;
                        destroy(pol, e, f, g);
                    }
                }
            }
#endif
        }
        unsigned coop = __ballot_sync(0xffffffffu, live && !serial);
        while (coop) {                                  // the whole warp, one edge at a time
            const int src = __ffs(coop) - 1;
            coop &= coop - 1;
#if GC_PEEL_PF
            if (coop) {   // TMA bulk L2 prefetch of the next edge's rows while this one is walked
                const int nx = __ffs(coop) - 1;
                const int64_t na0 = __shfl_sync(0xffffffffu, a0, nx), na1 = __shfl_sync(0xffffffffu, a1, nx);
                const int64_t nb0 = __shfl_sync(0xffffffffu, b0, nx), nb1 = __shfl_sync(0xffffffffu, b1, nx);
                if (lane == 0) {
                    const int64_t t0 = max(na0, na1 - 64);   // the walk's first chunks, from the row end
                    row_pf(A.sym_col, t0, na1);
                    row_pf(A.sym_eid, t0, na1);
                    if (nb1 - nb0 <= GC_PEEL_PF_MAX) row_pf(A.sym_col, nb0, nb1);   // the searched row, whole
                }
            }
#endif
            peel_one_warp<Pol>(A, pol, __shfl_sync(0xffffffffu, e, src), __shfl_sync(0xffffffffu, live, src),
                          __shfl_sync(0xffffffffu, a0, src), __shfl_sync(0xffffffffu, a1, src),
                          __shfl_sync(0xffffffffu, b0, src), __shfl_sync(0xffffffffu, b1, src), lane);
        }
    }
}


// ------------------------------------- grouped heavy edges (dense-core rounds) --
// When a dense core collapses, single rounds carry 10^6-10^7 frontier edges
// whose endpoints both have thousands of live neighbours (C5 level 2,496:
// rounds of 5-19 M edges, 2.8 s each with the per-edge search).  Such rounds
// group their heavy edges (shorter live row >= heavy_row) by pivot x, the
// endpoint with the longer row: a block stages N_live(x) once as a 32 KB
// rank-window bitmap, each warp streams the other endpoint's row of one heavy
// edge and probes it, and only the hits (the live triangles) search row x for
// the third edge's id.  Light edges keep the per-edge search.
constexpr int kGrpBits = 1 << 18;      // bitmap window (ranks)
constexpr int kGrpChunk = 1024;        // heavy edges per group at most

template <class Pol>
__global__ void k_split_heavy(PeelArgs A, Pol pol, int heavy_row, uint32_t* __restrict__ hkey,
                              int32_t* __restrict__ hval, int* __restrict__ hcount, int32_t* __restrict__ light,
                              int* __restrict__ lcount) {
    const int lane = threadIdx.x & 31;
    const int nfront = A.nfront_dev ? *A.nfront_dev : A.nfront;
    for (int i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; i0 < nfront; i0 += gridDim.x * blockDim.x) {
        const int i = i0 + lane;
        int e = -1, x = 0;
        bool heavy = false, lgt = false;
        if (i < nfront) {
            e = A.front[i];
            if (pol.live(e)) {
                const int a = A.dag_src[e], b = A.dag_col[e];
                const int la = A.live_len[a], lb = A.live_len[b];
                heavy = min(la, lb) >= heavy_row;
                lgt = !heavy;
                x = lb >= la ? b : a;
            }
        }
        const unsigned hb = __ballot_sync(0xffffffffu, heavy), lb2 = __ballot_sync(0xffffffffu, lgt);
        int hbase = 0, lbase = 0;
        if (lane == 0) {
            if (hb) hbase = atomicAdd(hcount, __popc(hb));
            if (lb2) lbase = atomicAdd(lcount, __popc(lb2));
        }
        hbase = __shfl_sync(0xffffffffu, hbase, 0);
        lbase = __shfl_sync(0xffffffffu, lbase, 0);
        const unsigned below = (1u << lane) - 1;
        if (heavy) {
            const int o = hbase + __popc(hb & below);
            hkey[o] = (uint32_t)x;
            hval[o] = e;
        }
        if (lgt) light[lbase + __popc(lb2 & below)] = e;
    }
}

__global__ void k_group_flags(const uint32_t* __restrict__ key, int nh, uint8_t* __restrict__ flag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x)
        flag[i] = (i == 0 || key[i] != key[i - 1] || i % kGrpChunk == 0) ? 1 : 0;
}

constexpr size_t kGrpSmem = kGrpBits / 8 + kGrpBits / 64 * 4 + 64;   // bitmap + prefix per 64 ranks

template <class Pol>
__global__ void __launch_bounds__(256, GC_GRP_MINB) k_peel_grouped(PeelArgs A, Pol pol, const uint32_t* __restrict__ key,
                                                         const int32_t* __restrict__ edges, int nh,
                                                         const int32_t* __restrict__ starts,
                                                         const int* __restrict__ ngroups) {
    // bits: every entry of the pivot row x (dead ones too), offset from its
    // first rank wb; pre[c]: entries below rank wb + 64 c, so the position of
    // a hit in row x -- and the third edge's id -- needs no search.
    extern __shared__ unsigned long long grp_smem[];
    unsigned long long* bits = grp_smem;
    uint32_t* pre = reinterpret_cast<uint32_t*>(bits + kGrpBits / 64);
    int* s_ok = reinterpret_cast<int*>(pre + kGrpBits / 64);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = *ngroups;
    for (int j = threadIdx.x; j < kGrpBits / 64; j += blockDim.x) bits[j] = 0ull;   // zero between groups
    __syncthreads();
    for (int gi = blockIdx.x; gi < G; gi += gridDim.x) {
        const int g0 = starts[gi], g1 = gi + 1 < G ? starts[gi + 1] : nh;
        const int x = (int)key[g0];
        const int64_t xb = A.sym_ptr[x];
        const int L = A.live_len[x];
        const int32_t wb = A.sym_col[xb];
        const int32_t span = A.sym_col[xb + L - 1] - wb;
        const bool ok = span < kGrpBits;
        if (ok) {
            for (int i = threadIdx.x; i < L; i += blockDim.x) {
                const uint32_t off = (uint32_t)(A.sym_col[xb + i] - wb);
                atomicOr(bits + (off >> 6), 1ull << (off & 63));
            }
            __syncthreads();
            // exclusive prefix of the chunk popcounts: 16 chunks per thread + a block scan
            const int nch = (span >> 6) + 1;
            const int c0 = threadIdx.x * (kGrpBits / 64 / 256);
            uint32_t loc = 0;
            if (c0 < nch)
                for (int c = c0; c < c0 + kGrpBits / 64 / 256; ++c) loc += __popcll(bits[c]);
            uint32_t inc = loc;
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += t;
            }
            if (lane == 31) s_ok[1 + warp] = (int)inc;
            __syncthreads();
            uint32_t base = inc - loc;
            for (int w = 0; w < warp; ++w) base += (uint32_t)s_ok[1 + w];
            if (c0 < nch)
                for (int c = c0; c < c0 + kGrpBits / 64 / 256; ++c) {
                    pre[c] = base;
                    base += __popcll(bits[c]);
                }
        }
        __syncthreads();
        for (int k = g0 + warp; k < g1; k += 8) {
            const int e = edges[k];
            const uint32_t live = pol.live(e);
            const int a = A.dag_src[e], b = A.dag_col[e];
            const int y = a == x ? b : a;
            const int64_t y0 = A.sym_ptr[y], y1 = y0 + A.live_len[y];
            if (!ok) {
                peel_one_warp(A, pol, e, live, y0, y1, xb, xb + L, lane);
                continue;
            }
            uint32_t found = 0;
            for (int64_t q = y0; q < y1 && found < live; q += 32) {
                const int64_t i = q + lane;
                bool tri = false;
                int f = -1, g = -1;
                if (i < y1) {
                    const uint32_t off = (uint32_t)(__ldg(A.sym_col + i) - wb);
                    const unsigned long long word = off < (uint32_t)kGrpBits ? bits[off >> 6] : 0ull;
                    if ((word >> (off & 63)) & 1ull) {
                        f = __ldg(A.sym_eid + i);
                        if (f != e && A.alive[f]) {
                            const uint32_t pos = pre[off >> 6] + __popcll(word & ((1ull << (off & 63)) - 1));
                            g = __ldg(A.sym_eid + xb + pos);
                            tri = A.alive[g] != 0;
                        }
                    }
                }
                found += __popc(__ballot_sync(0xffffffffu, tri));
                if (tri) destroy(pol, e, f, g);
            }
        }
        __syncthreads();
        if (ok)
            for (int i = threadIdx.x; i < L; i += blockDim.x)
                bits[(uint32_t)(A.sym_col[xb + i] - wb) >> 6] = 0ull;
        __syncthreads();
    }
}

// ---------------------------------------------- partitioned peel (§8(e) v1) --
// Edges (DAG positions) are owned in word-aligned contiguous ranges, one per
// rank; every rank keeps the replicated alive set and the exact support of
// the edges it owns.  Per round the removed set X travels as a bitmap
// (ncclAllGather of each owner's slice), every rank enumerates the destroyed
// triangles of the whole X and decrements only the survivors it owns.

// own slices at a level start, e in [lo, hi): X bit = alive && 0 < S < thr
// (the round's frontier), Z bit = alive && S == 0 < thr (in no live triangle:
// removed on every rank without enumeration), and min S over the owned
// alive edges left out (the empty-level skip)
__global__ void k_front_bits(const uint32_t* __restrict__ S, const uint8_t* __restrict__ alive, int64_t lo,
                             int64_t hi, uint32_t thr, uint32_t* __restrict__ xbits, uint32_t* __restrict__ zbits,
                             uint32_t* __restrict__ min_rest) {
    // lo is a multiple of 32: thread e's ballot is word e / 32
    uint32_t rest = 0xFFFFFFFFu;
    for (int64_t e = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < lo + (((hi - lo) + 31) & ~(int64_t)31);
         e += (int64_t)gridDim.x * blockDim.x) {
        const bool al = e < hi && alive[e];
        const uint32_t se = al ? S[e] : 0xFFFFFFFFu;
        const bool zero = al && se == 0 && thr > 0;
        const bool in = al && se > 0 && se < thr;
        if (al && !zero && !in) rest = min(rest, se);
        const unsigned wx = __ballot_sync(0xffffffffu, in);
        const unsigned wz = __ballot_sync(0xffffffffu, zero);
        if ((threadIdx.x & 31) == 0) {
            xbits[e >> 5] = wx;
            zbits[e >> 5] = wz;
        }
    }
    rest = __reduce_min_sync(0xffffffffu, rest);
    if ((threadIdx.x & 31) == 0 && rest != 0xFFFFFFFFu) atomicMin(min_rest, rest);
}

// the gathered zero-support edges leave (every rank): alive = 0, tau = level
__global__ void k_zero_finish(const uint32_t* __restrict__ zbits, int64_t nwords, uint8_t* __restrict__ alive,
                              int32_t* __restrict__ tau, int32_t level, unsigned long long* __restrict__ acc) {
    unsigned c = 0;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = zbits[w];
        c += __popc(x);
        while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            const int64_t e = w * 32 + b;
            alive[e] = 0;
            if (tau) tau[e] = level;
        }
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(acc, (unsigned long long)c);
}

// list of the set bits of bits[0, nwords) (order unspecified)
__global__ void k_bits_to_list(const uint32_t* __restrict__ bits, int64_t nwords, int32_t* __restrict__ list,
                               int* __restrict__ count) {
    const int lane = threadIdx.x & 31;
    for (int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~(int64_t)31; w0 < nwords;
         w0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = w0 + lane;
        uint32_t x = w < nwords ? bits[w] : 0u;
        const int c = __popc(x);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        int base = 0;
        if (lane == 31 && tot) base = atomicAdd(count, tot);
        base = __shfl_sync(0xffffffffu, base, 31) + incl - c;
        while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            list[base++] = (int32_t)(w * 32 + b);
        }
    }
}

// list entries (indices within a slice) += the slice's first edge
__global__ void k_offset_list(int32_t* __restrict__ list, const int* __restrict__ n_dev, int32_t off) {
    const int n = *n_dev;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) list[i] += off;
}

__global__ void k_u64_to_u32(const unsigned long long* __restrict__ a, uint32_t* __restrict__ b) {
    if (threadIdx.x == 0) *b = *a > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)*a;
}

// received decrements (NCCL partitioned peel): apply those of this rank's
// edges [lo, hi) to its support copy; a crossing sets the next X bit
__global__ void k_apply_decrements(const int32_t* __restrict__ in, int64_t n, int64_t lo, int64_t hi,
                                   uint32_t* __restrict__ S, uint32_t thr, uint32_t* __restrict__ nbits) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int f = in[i];
        if (f >= lo && f < hi && atomicSub(S + f, 1u) == thr) atomicOr(nbits + (f >> 5), 1u << (f & 31));
    }
}

// sort key of a frontier edge: its endpoint with the longer live row (the row
// the per-edge search probes), so edges probing the same row run together
__global__ void k_pivot_keys(const int32_t* __restrict__ front, int nf, const int32_t* __restrict__ dag_src,
                             const int32_t* __restrict__ dag_col, const int32_t* __restrict__ live_len,
                             uint32_t* __restrict__ keys) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
        const int e = front[i];
        const int a = dag_src[e], b = dag_col[e];
        keys[i] = (uint32_t)(live_len[a] > live_len[b] ? a : b);
    }
}

// End of a round: the frontier (its size on the device) leaves the alive set
// (tau = level in a decomposition); also counts the removed edges and the
// non-empty rounds
__global__ void k_finish_round_dev(const int32_t* __restrict__ front, const int* __restrict__ nfront_dev,
                                   uint8_t* __restrict__ alive, int32_t* __restrict__ tau, int32_t level,
                                   unsigned long long* __restrict__ acc) {
    const int nfront = *nfront_dev;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nfront; i += gridDim.x * blockDim.x) {
        int e = front[i];
        alive[e] = 0;
        if (tau) tau[e] = level;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && nfront > 0) {
        acc[0] += (unsigned long long)nfront;
        acc[1] += 1ULL;
    }
}

// mask from the canonical supports when the peel ran no round: it then only
// removed zero-support edges (at the level scan), so alive = (S >= 1)
// mask[i] = S[i] >= thr, and the number of kept edges (any order of S)
__global__ void k_mask_from_support(const uint32_t* __restrict__ S, int64_t m, uint32_t thr,
                                    uint8_t* __restrict__ out, unsigned long long* __restrict__ kept) {
    unsigned c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const bool in = S[i] >= thr;
        out[i] = in;
        c += in;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(kept, (unsigned long long)c);
}

// ---- k-truss byte-model terms (GC_OPT_WORK_STATS)
// alive degree of every vertex at the peel start (every edge alive)
__global__ void k_vdeg_init(const int64_t* __restrict__ dag_ptr, const int64_t* __restrict__ in_ptr, int64_t n,
                            int32_t* __restrict__ vdeg) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
        vdeg[x] = (int32_t)((dag_ptr[x + 1] - dag_ptr[x]) + (in_ptr[x + 1] - in_ptr[x]));
}

// acc += sum over the round's frontier edges e = (a,b) with S(e) > 0 of
// min(vdeg[a], vdeg[b]) (degrees at the round start)
__global__ void k_round_summin(const int32_t* __restrict__ front, const int* __restrict__ nfront_dev,
                               const uint32_t* __restrict__ S, const int32_t* __restrict__ dag_src,
                               const int32_t* __restrict__ dag_col, const int32_t* __restrict__ vdeg,
                               unsigned long long* __restrict__ acc) {
    const int nf = *nfront_dev;
    unsigned long long sum = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
        const int e = front[i];
        if (S[e] > 0) sum += (unsigned long long)min(vdeg[dag_src[e]], vdeg[dag_col[e]]);
    }
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0 && sum) atomicAdd(acc, sum);
}

// the removed edges leave their endpoints' alive degrees
__global__ void k_round_vdeg(const int32_t* __restrict__ list, const int* __restrict__ n_dev,
                             const int32_t* __restrict__ dag_src, const int32_t* __restrict__ dag_col,
                             int32_t* __restrict__ vdeg) {
    const int nl = *n_dev;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) {
        const int e = list[i];
        atomicSub(vdeg + dag_src[e], 1);
        atomicSub(vdeg + dag_col[e], 1);
    }
}

__global__ void k_sum_u32(const uint32_t* __restrict__ a, int64_t m, unsigned long long* __restrict__ acc) {
    unsigned long long sum = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        sum += a[i];
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0 && sum) atomicAdd(acc, sum);
}


}  // namespace

int build_sym(gc_ctx* c) {
    if (c->sym_ready) return GC_OK;
    const int64_t n = c->n, m = c->m;
    GC_TRY(ensure(c, c->sym_ptr, (size_t)(n + 1) * 8));
    GC_TRY(ensure(c, c->sym_col, (size_t)2 * m * 4 + 64));   // +64: 16-byte aligned bulk prefetches
    GC_TRY(ensure(c, c->sym_eid, (size_t)2 * m * 4 + 64));
    GC_TRY(ensure(c, c->live_len, (size_t)n * 4));
    GC_TRY(ensure(c, c->long_rows, (size_t)n * 4));
    GC_LAUNCH(c, k_sym_ptr, grid_for(n + 1), kThreads, 0, c->dag_ptr.as<int64_t>(), c->in_ptr.as<int64_t>(), n,
              c->sym_ptr.as<int64_t>());
    int* cnt = reinterpret_cast<int*>(c->scal.as<char>() + 232);
    GC_CUDA(c, cudaMemsetAsync(cnt, 0, sizeof(int), c->stream));
    if (n > 0)
        GC_LAUNCH(c, k_long_rows, grid_for(n), kThreads, 0, c->sym_ptr.as<int64_t>(), n, c->long_rows.as<int32_t>(),
                  cnt);
    GC_TRY(read_small(c, c->hpin, cnt, sizeof(int)));
    GC_TRY(sync(c));
    c->nlong = *static_cast<int*>(c->hpin);
    c->sym_ready = true;
    c->sym_dirty = true;
    return GC_OK;
}

// (Re)fill the symmetric rows from the DAG: every entry live, full lengths.
static int sym_refill(gc_ctx* c) {
    const int64_t n = c->n, m = c->m;
    if (m > 0)
        GC_LAUNCH(c, k_sym_fill, grid_for(m), kThreads, 0, c->in_src.as<int32_t>(), c->in_dst.as<int32_t>(),
                  c->in_pos.as<int32_t>(), c->dag_src.as<int32_t>(), c->dag_col.as<int32_t>(),
                  c->dag_ptr.as<int64_t>(), c->in_ptr.as<int64_t>(), m, c->sym_col.as<int32_t>(),
                  c->sym_eid.as<int32_t>());
    if (n > 0)
        GC_LAUNCH(c, k_live_len_init, grid_for(n), kThreads, 0, c->sym_ptr.as<int64_t>(), n,
                  c->live_len.as<int32_t>());
    c->sym_dirty = false;
    return GC_OK;
}

// Drop dead entries from the rows once the live edge count has fallen to
// (compact_div - 1) / compact_div of what it was at the last compaction (or the start): the
// searches re-read row sectors from DRAM, so denser rows pay (C4 / C5 decomposition kernel +
// scan + compaction 1.55 / 19.0 s at 1/2, 1.44 / 18.1 s at 4/5).
static int maybe_compact(gc_ctx* c) {
    if (!c->rows_live) return GC_OK;
    // compact once the live edges fall to (v - 1) / v of the last compaction, v = compact_div
    // in a decomposition (many levels follow to repay it); a single k-truss keeps v <= 2
    const int64_t v = c->decomp_running ? c->compact_div : std::min(c->compact_div, 2);
    if (v <= 1 || c->m_alive_h <= 0 || c->m_alive_h * v > c->compact_at * (v - 1)) return GC_OK;
    const int64_t n = c->n, m = c->m;
    GC_TRY(record(c, 12));
    GC_LAUNCH(c, k_row_compact_warp, grid_for(n * 32), kThreads, 0, c->sym_ptr.as<int64_t>(),
              c->live_len.as<int32_t>(), c->sym_col.as<int32_t>(), c->sym_eid.as<int32_t>(), c->alive.as<uint8_t>(), n);
    if (c->nlong > 0)
        GC_LAUNCH(c, k_row_compact_block, std::min(c->nlong, 148 * 8), 256, 0, c->long_rows.as<int32_t>(), c->nlong,
                  c->sym_ptr.as<int64_t>(), c->live_len.as<int32_t>(), c->sym_col.as<int32_t>(),
                  c->sym_eid.as<int32_t>(), c->alive.as<uint8_t>());
    int* cnt = reinterpret_cast<int*>(c->scal.as<char>() + 232);
    GC_CUDA(c, cudaMemsetAsync(cnt, 0, sizeof(int), c->stream));
    GC_LAUNCH(c, k_alive_list, grid_for(m), kThreads, 0, c->alive.as<uint8_t>(), m, c->alist.as<int32_t>(), cnt);
    GC_TRY(record(c, 13));
    GC_TRY(sync(c));
    c->stats.compact_ms += elapsed(c, 12, 13);
    c->alist_n = c->m_alive_h;
    c->compact_at = c->m_alive_h;
    c->sym_dirty = true;              // the next peel call refills the rows
    c->stats.compactions++;
    return GC_OK;
}

// Symmetric rows are needed only once a round has triangles to destroy (the
// k = 3 peel removes its zero-support edges during the scan and never needs
// them): built / refilled on first use within a peel call.
static int ensure_rows(gc_ctx* c) {
    if (c->rows_live) return GC_OK;
    GC_TRY(build_sym(c));
    if (c->sym_dirty) GC_TRY(sym_refill(c));
    c->rows_live = true;
    return GC_OK;
}

// k_peel for a round of nf frontier edges (nf < 0: known only on the device)
template <class Pol>
static int launch_peel(gc_ctx* c, int blocks, const PeelArgs& A, const Pol& pol, int64_t nf) {
    if (nf < 0 || nf >= c->peel_big) {
        GC_LAUNCH(c, (k_peel<Pol, 1>), blocks, 256, 0, A, pol);
    } else {
        GC_LAUNCH(c, (k_peel<Pol, 8>), blocks, 256, 0, A, pol);
    }
    return GC_OK;
}

// One peel round over the frontier list.
template <class Pol>
static int peel_round(gc_ctx* c, const int32_t* front, int nf, const Pol& pol) {
    PeelArgs A{front, nf, nullptr, c->dag_src.as<int32_t>(), c->dag_col.as<int32_t>(), c->sym_ptr.as<int64_t>(),
               c->live_len.as<int32_t>(), c->sym_col.as<int32_t>(), c->sym_eid.as<int32_t>(),
               c->alive.as<uint8_t>()};
    const int blocks = (int)std::min<int64_t>(((int64_t)nf * 32 + 255) / 256, 148 * 8);
    return launch_peel(c, blocks, A, pol, nf);
}


// A dense-core round: light frontier edges by the per-edge search, heavy ones
// grouped by pivot (k_peel_grouped).  front / nf on the host.
template <class Pol>
static int peel_round_grouped(gc_ctx* c, const int32_t* front, int nf, const Pol& pol) {
    GC_TRY(ensure(c, c->grp_keys, (size_t)nf * 4 * 2));
    GC_TRY(ensure(c, c->grp_vals, (size_t)nf * 4 * 2));
    GC_TRY(ensure(c, c->grp_starts, (size_t)nf * 4 + 4));
    GC_TRY(ensure(c, c->grp_flags, (size_t)nf + 4));
    GC_TRY(ensure(c, c->grp_light, (size_t)nf * 4 + 4));
    uint32_t* k0 = c->grp_keys.as<uint32_t>();
    uint32_t* k1 = k0 + nf;
    int32_t* v0 = c->grp_vals.as<int32_t>();
    int32_t* v1 = v0 + nf;
    int* cnts = reinterpret_cast<int*>(c->scal.as<char>() + 304);   // heavy, light, groups
    GC_CUDA(c, cudaMemsetAsync(cnts, 0, 3 * sizeof(int), c->stream));
    PeelArgs A{front, nf, nullptr, c->dag_src.as<int32_t>(), c->dag_col.as<int32_t>(), c->sym_ptr.as<int64_t>(),
               c->live_len.as<int32_t>(), c->sym_col.as<int32_t>(), c->sym_eid.as<int32_t>(),
               c->alive.as<uint8_t>()};
    GC_LAUNCH(c, k_split_heavy<Pol>, grid_for(nf), kThreads, 0, A, pol, c->group_heavy, k0, v0, cnts,
              c->grp_light.as<int32_t>(), cnts + 1);
    PeelArgs Lt = A;
    Lt.front = c->grp_light.as<int32_t>();
    Lt.nfront = 0;
    Lt.nfront_dev = cnts + 1;
    GC_TRY(launch_peel(c, 148 * 8, Lt, pol, -1));
    int32_t* h = static_cast<int32_t*>(c->hpin);
    GC_TRY(read_small(c, h + 8, cnts, sizeof(int)));
    GC_TRY(sync(c));
    const int nh = h[8];
    if (nh == 0) return GC_OK;
    const int kbits = std::max(1, ceil_log2_u64((uint64_t)c->n));
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, nh, 0, kbits, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, k0, k1, v0, v1, nh, 0, kbits, c->stream));
    GC_LAUNCH(c, k_group_flags, grid_for(nh), kThreads, 0, k1, nh, c->grp_flags.as<uint8_t>());
    thrust::counting_iterator<int32_t> iota(0);
    tmp = 0;
    GC_CUDA(c, cub::DeviceSelect::Flagged(nullptr, tmp, iota, c->grp_flags.as<uint8_t>(), c->grp_starts.as<int32_t>(),
                                          cnts + 2, nh, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, iota, c->grp_flags.as<uint8_t>(),
                                          c->grp_starts.as<int32_t>(), cnts + 2, nh, c->stream));
    c->stats.lib_launches += 4 + (kbits + 7) / 8;
    GC_CUDA(c, cudaFuncSetAttribute(k_peel_grouped<Pol>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGrpSmem));
    GC_LAUNCH(c, k_peel_grouped<Pol>, 148 * 4, 256, kGrpSmem, A, pol, k1, v1, nh, c->grp_starts.as<int32_t>(),
              cnts + 2);
    return GC_OK;
}

// A big frontier (nf known on the host) sorted by the endpoint whose live row
// the per-edge search probes (GC_OPT_SORT_FRONT): warps that search the same
// hub row run close together and find its sectors in L2.
static int sort_frontier(gc_ctx* c, int32_t* front, int nf) {
    GC_TRY(ensure(c, c->grp_keys, (size_t)nf * 4 * 2));
    GC_TRY(ensure(c, c->grp_vals, (size_t)nf * 4));
    uint32_t* k0 = c->grp_keys.as<uint32_t>();
    uint32_t* k1 = k0 + nf;
    int32_t* v1 = c->grp_vals.as<int32_t>();
    GC_LAUNCH(c, k_pivot_keys, grid_for(nf), kThreads, 0, front, nf, c->dag_src.as<int32_t>(), c->dag_col.as<int32_t>(),
              c->live_len.as<int32_t>(), k0);
    const int kbits = std::max(1, ceil_log2_u64((uint64_t)c->n));
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, front, v1, nf, 0, kbits, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, k0, k1, front, v1, nf, 0, kbits, c->stream));
    c->stats.lib_launches += 2 + (kbits + 7) / 8;
    GC_CUDA(c, cudaMemcpyAsync(front, v1, (size_t)nf * 4, cudaMemcpyDeviceToDevice, c->stream));
    return GC_OK;
}

// Work stats (GC_OPT_WORK_STATS): the edges of `gone` (count on the device)
// leave the alive degrees, then the next round's frontier `next` adds its
// min-degree term (either list may be null).
static int work_round(gc_ctx* c, const int32_t* next, const int* next_n, const int32_t* gone, const int* gone_n) {
    if (gone)
        GC_LAUNCH(c, k_round_vdeg, 148 * 4, kThreads, 0, gone, gone_n, c->dag_src.as<int32_t>(),
                  c->dag_col.as<int32_t>(), c->vdeg.as<int32_t>());
    if (next)
        GC_LAUNCH(c, k_round_summin, 148 * 4, kThreads, 0, next, next_n, c->sup.as<uint32_t>(),
                  c->dag_src.as<int32_t>(), c->dag_col.as<int32_t>(), c->vdeg.as<int32_t>(),
                  reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 672));
    return GC_OK;
}

// Peel at threshold thr = k - 2 starting from the current alive set / S.
// level >= 0: write tau = level for removed edges.  Returns removed count.
#ifndef GC_BATCH_MAX_FRONT
#define GC_BATCH_MAX_FRONT 16384
#endif
constexpr int kBatchMaxFront = GC_BATCH_MAX_FRONT;

// *next_thr (when non-null): with an empty frontier nothing but S = 0 edges
// left, so no S changed and every threshold up to min S over the survivors
// finds an empty frontier too -- the smallest threshold worth scanning next
// (0: unknown, the frontier was not empty).  The decomposition jumps there
// (C5: 757 non-empty levels of 2,873).
static int peel_level(gc_ctx* c, uint32_t thr, int32_t level, int32_t* round, int64_t* removed,
                      uint32_t* next_thr) {
    const int64_t m = c->m;
    // diagnostics: GC_PROFILE_LEVEL=<k-1> brackets that level with the CUDA
    // profiler start/stop (ncu --profile-from-start off)
    static const int prof_level = getenv("GC_PROFILE_LEVEL") ? atoi(getenv("GC_PROFILE_LEVEL")) : -2;
    struct ProfScope {
        bool on;
        ~ProfScope() { if (on) cudaProfilerStop(); }
    } prof{prof_level == level};
    if (prof.on) cudaProfilerStart();
    int* cnt = reinterpret_cast<int*>(c->scal.as<char>() + 224);
    int32_t* h = static_cast<int32_t*>(c->hpin);
    *removed = 0;
    GC_TRY(maybe_compact(c));
    GC_CUDA(c, cudaMemsetAsync(cnt, 0, 2 * sizeof(int), c->stream));
    const int32_t* list = c->alist_n >= 0 ? c->alist.as<int32_t>() : nullptr;
    const int64_t len = c->alist_n >= 0 ? c->alist_n : m;
    GC_TRY(record(c, 10));
    unsigned long long* zrem = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 240);
    uint32_t* min_rest = reinterpret_cast<uint32_t*>(c->scal.as<char>() + 320);
    GC_CUDA(c, cudaMemsetAsync(zrem, 0, 8, c->stream));
    GC_CUDA(c, cudaMemsetAsync(min_rest, 0xFF, 4, c->stream));
    const bool ws = c->work_stats != 0;
    int* zc = reinterpret_cast<int*>(c->scal.as<char>() + 688);
    if (ws) GC_CUDA(c, cudaMemsetAsync(zc, 0, sizeof(int), c->stream));
    GC_LAUNCH(c, k_frontier_scan, grid_for(len), kThreads, 0, c->sup.as<uint32_t>(), c->alive.as<uint8_t>(), list,
              len, thr, *round, c->front_a.as<int32_t>(), cnt,
              level >= 0 ? c->tau.as<int32_t>() : nullptr, level, zrem, min_rest,
              ws ? c->zlist.as<int32_t>() : nullptr, zc);
    if (ws) {
        // round 1's X = the scan's frontier plus the zero-support edges it
        // removed on the spot: its term uses the degrees before either leaves
        GC_TRY(work_round(c, c->front_a.as<int32_t>(), cnt, nullptr, nullptr));
        GC_TRY(work_round(c, nullptr, nullptr, c->zlist.as<int32_t>(), zc));
    }
    GC_TRY(record(c, 11));
    GC_TRY(read_small(c, h, cnt, sizeof(int)));
    GC_TRY(read_small(c, h + 2, zrem, 8));
    GC_TRY(read_small(c, h + 4, min_rest, 4));
    GC_TRY(sync(c));
    c->stats.scan_ms += elapsed(c, 10, 11);
    {
        const int64_t z = *reinterpret_cast<int64_t*>(h + 2);   // removed on the spot (S = 0)
        *removed += z;
        c->m_alive_h -= z;
    }
    int nf = h[0];
    if (next_thr) {
        const uint32_t mr = static_cast<uint32_t>(h[4]);   // 0xFFFFFFFF: no survivor
        *next_thr = nf > 0 ? 0u : (mr == 0xFFFFFFFFu ? 0u : mr + 1);
    }
    if (nf > 0) GC_TRY(ensure_rows(c));
    // Rounds are enqueued in batches without a host round trip: each round's
    // kernels read the frontier size on the device (an empty frontier makes a
    // round a no-op), and the host looks at the next frontier size only after
    // each batch (batch length 2, 4, ..., 16 rounds within a level).
    int32_t* lists[2] = {c->front_a.as<int32_t>(), c->front_b.as<int32_t>()};
    int* counts[2] = {cnt, cnt + 1};
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 256);   // removed, rounds
    GC_CUDA(c, cudaMemsetAsync(acc, 0, 16, c->stream));
    const int64_t alive0 = c->m_alive_h;
    int cur = 0, batch = c->trace > 1 ? 1 : 2;   // GC_PEEL_TRACE=2: one round per batch (per-round trace)
    unsigned long long done[2] = {0, 0};
    int last_nf = nf;
    while (nf > 0) {
        if (c->group_peel > 0 && nf >= c->group_peel && c->stats.max_degree >= c->group_heavy) {
            // a dense-core round with a host round trip: heavy edges grouped by pivot
            const int nxt = cur ^ 1;
            GC_TRY(record(c, 8));
            GC_CUDA(c, cudaMemsetAsync(counts[nxt], 0, sizeof(int), c->stream));
            PolicySingle pol{c->alive.as<uint8_t>(), c->sup.as<uint32_t>(), thr, *round, lists[nxt], counts[nxt]};
            GC_TRY(peel_round_grouped(c, lists[cur], nf, pol));
            GC_LAUNCH(c, k_finish_round_dev, 148 * 4, kThreads, 0, lists[cur], counts[cur], c->alive.as<uint8_t>(),
                      level >= 0 ? c->tau.as<int32_t>() : nullptr, level, acc);
            if (ws) GC_TRY(work_round(c, lists[nxt], counts[nxt], lists[cur], counts[cur]));
            GC_TRY(record(c, 9));
            ++*round;
            cur = nxt;
            GC_TRY(read_small(c, h, counts[cur], sizeof(int)));
            GC_TRY(read_small(c, h + 2, acc, 16));
            GC_TRY(sync(c));
            c->stats.peel_kernel_ms += elapsed(c, 8, 9);
            memcpy(done, h + 2, 16);
            if (c->trace)
                fprintf(stderr, "peel-trace level %d grouped nf %d rounds %llu removed %llu ms %.4f\n", level, nf,
                        done[1], done[0], elapsed(c, 8, 9));
            c->m_alive_h = alive0 - (int64_t)done[0];
            nf = h[0];
            if (nf > 0) GC_TRY(maybe_compact(c));
            continue;
        }
        GC_TRY(record(c, 8));
        for (int r = 0; r < batch; ++r) {
            const int nxt = cur ^ 1;
            GC_CUDA(c, cudaMemsetAsync(counts[nxt], 0, sizeof(int), c->stream));
            PolicySingle pol{c->alive.as<uint8_t>(), c->sup.as<uint32_t>(), thr, *round, lists[nxt], counts[nxt]};
            if (r == 0 && c->sort_front > 0 && nf >= c->sort_front) GC_TRY(sort_frontier(c, lists[cur], nf));
            PeelArgs A{lists[cur], 0, counts[cur], c->dag_src.as<int32_t>(), c->dag_col.as<int32_t>(),
                       c->sym_ptr.as<int64_t>(), c->live_len.as<int32_t>(), c->sym_col.as<int32_t>(),
                       c->sym_eid.as<int32_t>(), c->alive.as<uint8_t>()};
            GC_TRY(launch_peel(c, 148 * 8, A, pol, r == 0 ? (int64_t)nf : 0));   // later rounds of a batch are small
            GC_LAUNCH(c, k_finish_round_dev, 148 * 4, kThreads, 0, lists[cur], counts[cur], c->alive.as<uint8_t>(),
                      level >= 0 ? c->tau.as<int32_t>() : nullptr, level, acc);
            if (ws) GC_TRY(work_round(c, lists[nxt], counts[nxt], lists[cur], counts[cur]));
            ++*round;
            cur = nxt;
        }
        GC_TRY(record(c, 9));
        GC_TRY(read_small(c, h, counts[cur], sizeof(int)));
        GC_TRY(read_small(c, h + 2, acc, 16));
        GC_TRY(sync(c));
        c->stats.peel_kernel_ms += elapsed(c, 8, 9);
        memcpy(done, h + 2, 16);
        if (c->trace)
            fprintf(stderr, "peel-trace level %d batch %d nf %d rounds %llu removed %llu ms %.4f\n", level, batch, nf,
                    done[1], done[0], elapsed(c, 8, 9));
        c->m_alive_h = alive0 - (int64_t)done[0];
        nf = h[0];
        if (nf > 0) GC_TRY(maybe_compact(c));
        // Batches only while the frontier is small and not growing: a dense
        // core's collapse (frontiers growing 10^4 -> 10^7 within a few rounds)
        // runs a round per host check, so big rounds take the grouped path and
        // the row compaction as soon as the live edges halve (C5 kernel
        // 29.7 -> 26.8 s against blind batches of 16).
        if (c->trace < 2) batch = (nf >= kBatchMaxFront || nf > last_nf) ? 1 : std::min(batch * 2, 16);
        last_nf = nf;
    }
    *removed += (int64_t)done[0];
    c->stats.peel_rounds += (int64_t)done[1];
    ++*round;   // fresh stamp for the next level's scan
    return GC_OK;
}

// ---- partitioned peel (multi-GPU v1; loopback virtual ranks on one GPU)
static int peel_parts(const gc_ctx* c) {
    if (c->nccl) return c->nranks;            // a real communicator (one rank included)
    if (c->loop_parts > 1) return c->loop_parts;
    return c->peel_part ? 1 : 0;   // 0: single-GPU frontier-list peeler
}

static int64_t part_words(const gc_ctx* c, int P) { return ((c->m + 31) / 32 + P - 1) / P; }

static uint32_t* part_support(gc_ctx* c, int r) {
    if (c->loop_parts > 1) return c->sup_parts.as<uint32_t>() + (size_t)r * c->m;
    return c->sup.as<uint32_t>();
}

// NCCL rounds of the partitioned peel (host-driven).  Per round: this
// rank's slice of the gathered X is its frontier; it is cut into chunks of at
// most K edges so a chunk's decrements of other ranks' edges fit the send
// list (an X edge has S < thr, so it destroys fewer than thr triangles:
// at most 2 (thr - 1) decrements); the chunk count is the ranks' maximum
// (every rank issues the same collectives).  Per chunk: enumerate, allgather
// the list sizes, allgatherv the lists, apply the received ones this rank
// owns.  Then every rank removes the whole X and the next X is allgathered.
static int peel_rounds_nccl(gc_ctx* c, uint32_t thr, int32_t level, int nf, int64_t* removed, uint32_t* xb,
                            uint32_t* nb) {
    const int64_t m = c->m;
    const int P = c->nranks, me = c->rank;
    const int64_t W = part_words(c, P);
    const int64_t lo = std::min<int64_t>(m, (int64_t)me * W * 32), hi = std::min<int64_t>(m, (int64_t)(me + 1) * W * 32);
    int* cnt = reinterpret_cast<int*>(c->scal.as<char>() + 224);
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 256);
    unsigned long long* out_n = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 696);
    uint32_t* share = reinterpret_cast<uint32_t*>(c->scal.as<char>() + 704);   // P <= 64 u32 (704..960)
    int32_t* h = static_cast<int32_t*>(c->hpin);
    int32_t* own = c->front_a.as<int32_t>();
    int32_t* all = c->front_b.as<int32_t>();
    int32_t* tau = level >= 0 ? c->tau.as<int32_t>() : nullptr;
    const int64_t cap = std::max<int64_t>(1 << 20, std::min<int64_t>(m, (int64_t)1 << 26));
    GC_TRY(ensure(c, c->dec_out, (size_t)cap * 4));
    GC_TRY(ensure(c, c->dec_in, (size_t)cap * P * 4));
    const int64_t K = std::max<int64_t>(1, cap / (2 * (int64_t)std::max<uint32_t>(thr, 1)));
    const int64_t z = *removed, alive0 = c->m_alive_h;
    unsigned long long done[2] = {0, 0};
    while (nf > 0) {
        GC_TRY(record(c, 8));
        GC_CUDA(c, cudaMemsetAsync(nb, 0, (size_t)P * W * 4, c->stream));
        // own frontier, and the largest one over the ranks
        GC_CUDA(c, cudaMemsetAsync(cnt, 0, sizeof(int), c->stream));
        GC_LAUNCH(c, k_bits_to_list, grid_for(W), kThreads, 0, xb + (size_t)me * W, W, own, cnt);
        GC_LAUNCH(c, k_offset_list, grid_for(W * 32), kThreads, 0, own, cnt, (int32_t)(me * W * 32));
        GC_CUDA(c, cudaMemcpyAsync(share, cnt, 4, cudaMemcpyDeviceToDevice, c->stream));
        GC_TRY(allreduce_max_u32(c, share, 1));
        GC_TRY(read_small(c, h, cnt, 4));
        GC_TRY(read_small(c, h + 1, share, 4));
        GC_TRY(sync(c));
        const int64_t n_own = h[0], n_max = (uint32_t)h[1];
        const int64_t chunks = (n_max + K - 1) / K;
        for (int64_t ch = 0; ch < chunks; ++ch) {
            const int64_t i0 = std::min(n_own, ch * K), i1 = std::min(n_own, (ch + 1) * K);
            GC_CUDA(c, cudaMemsetAsync(out_n, 0, 8, c->stream));
            if (i1 > i0) {
                PolicyPart pol{xb, c->sup.as<uint32_t>(), 0, W * 32, me, thr, nb, c->dec_out.as<int32_t>(), out_n, cap};
                PeelArgs A{own + i0, (int)(i1 - i0), nullptr, c->dag_src.as<int32_t>(), c->dag_col.as<int32_t>(),
                           c->sym_ptr.as<int64_t>(), c->live_len.as<int32_t>(), c->sym_col.as<int32_t>(),
                           c->sym_eid.as<int32_t>(), c->alive.as<uint8_t>()};
                const int blocks = (int)std::min<int64_t>(((i1 - i0) * 32 + 255) / 256, 148 * 8);
                GC_TRY(launch_peel(c, blocks, A, pol, i1 - i0));
            }
            // sizes of every rank's send list, then the lists
            GC_LAUNCH(c, k_u64_to_u32, 1, 32, 0, out_n, share + me);   // saturates past 2^32 - 1
            GC_TRY(allgather_u32(c, share + me, share, 1));
            GC_TRY(read_small(c, h, share, (size_t)P * 4));
            GC_TRY(sync(c));
            int64_t counts[64], offs[64], tot = 0;
            for (int r = 0; r < P; ++r) {
                counts[r] = (uint32_t)h[r];
                offs[r] = tot;
                tot += counts[r];
            }
            // every rank sees every count, so all of them stop together (cannot happen: K bounds the lists)
            for (int r = 0; r < P; ++r)
                if (counts[r] > cap) return fail(c, GC_ERR_RANGE, "partitioned peel: decrement list overflow");
            if (tot > 0) {
                GC_TRY(allgatherv_i32(c, c->dec_out.as<int32_t>(), c->dec_in.as<int32_t>(), counts, offs));
                GC_LAUNCH(c, k_apply_decrements, grid_for(tot), kThreads, 0, c->dec_in.as<int32_t>(), tot, lo, hi,
                          c->sup.as<uint32_t>(), thr, nb);
            }
        }
        // every rank removes the whole X; the next X is gathered
        GC_CUDA(c, cudaMemsetAsync(cnt + 1, 0, sizeof(int), c->stream));
        GC_LAUNCH(c, k_bits_to_list, grid_for(P * W), kThreads, 0, xb, P * W, all, cnt + 1);
        GC_LAUNCH(c, k_finish_round_dev, 148 * 4, kThreads, 0, all, cnt + 1, c->alive.as<uint8_t>(), tau, level, acc);
        std::swap(xb, nb);
        GC_TRY(allgather_u32(c, xb + (size_t)me * W, xb, (size_t)W));
        GC_CUDA(c, cudaMemsetAsync(cnt, 0, sizeof(int), c->stream));
        GC_LAUNCH(c, k_bits_to_list, grid_for(P * W), kThreads, 0, xb, P * W, all, cnt);
        GC_TRY(record(c, 9));
        GC_TRY(read_small(c, h, cnt, sizeof(int)));
        GC_TRY(read_small(c, h + 2, acc, 16));
        GC_TRY(sync(c));
        c->stats.peel_kernel_ms += elapsed(c, 8, 9);
        memcpy(done, h + 2, 16);
        nf = h[0];
        c->m_alive_h = alive0 - (int64_t)done[0];
        if (nf > 0) GC_TRY(maybe_compact(c));
    }
    *removed = z + (int64_t)done[0];
    c->stats.peel_rounds += (int64_t)done[1];
    return GC_OK;
}

// One level of the partitioned peel.  At the level start each owner scans
// its range into the frontier bitmap X and the zero-support bitmap Z; both
// are allgathered, Z's edges leave on every rank without enumeration (they
// lie in no live triangle), and min S over the edges left out is combined
// (ncclAllReduce min) for the empty-level skip.  Rounds then run in
// device-side batches like the single-rank peeler: each round lists the
// gathered X, enumerates its destroyed triangles (owner-only decrements;
// crossings set bits of the next X), removes X and allgathers the next X,
// with no host round trip inside a batch; the host reads the next frontier
// size after each batch.  Every rank sees the same gathered bitmaps, so
// every rank takes the same batch decisions and issues the same collectives.
static int peel_level_part(gc_ctx* c, uint32_t thr, int32_t level, int64_t* removed, uint32_t* next_thr) {
    const int64_t m = c->m;
    const int P = peel_parts(c);
    const int64_t W = part_words(c, P);
    const bool nccl = c->nccl != nullptr;
    const int r_begin = nccl ? c->rank : 0, r_end = nccl ? c->rank + 1 : P;
    int* cnt = reinterpret_cast<int*>(c->scal.as<char>() + 224);      // two frontier counts
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 256);   // removed, rounds
    unsigned long long* zrem = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 240);
    uint32_t* min_rest = reinterpret_cast<uint32_t*>(c->scal.as<char>() + 320);
    int32_t* h = static_cast<int32_t*>(c->hpin);
    uint32_t* xb = c->xbits.as<uint32_t>();
    uint32_t* nb = c->nbits.as<uint32_t>();
    uint32_t* zb = c->zbits.as<uint32_t>();
    int32_t* lists[2] = {c->front_a.as<int32_t>(), c->front_b.as<int32_t>()};
    int* counts[2] = {cnt, cnt + 1};
    int32_t* tau = level >= 0 ? c->tau.as<int32_t>() : nullptr;
    *removed = 0;
    auto lo_of = [&](int r) { return std::min<int64_t>(m, (int64_t)r * W * 32); };
    auto hi_of = [&](int r) { return std::min<int64_t>(m, (int64_t)(r + 1) * W * 32); };
    GC_TRY(maybe_compact(c));
    GC_TRY(record(c, 10));
    GC_CUDA(c, cudaMemsetAsync(xb, 0, (size_t)P * W * 4, c->stream));
    GC_CUDA(c, cudaMemsetAsync(zb, 0, (size_t)P * W * 4, c->stream));
    GC_CUDA(c, cudaMemsetAsync(min_rest, 0xFF, 4, c->stream));
    GC_CUDA(c, cudaMemsetAsync(zrem, 0, 8, c->stream));
    GC_CUDA(c, cudaMemsetAsync(acc, 0, 16, c->stream));
    GC_CUDA(c, cudaMemsetAsync(cnt, 0, 2 * sizeof(int), c->stream));
    for (int r = r_begin; r < r_end; ++r)
        if (hi_of(r) > lo_of(r))
            GC_LAUNCH(c, k_front_bits, grid_for(hi_of(r) - lo_of(r)), kThreads, 0, part_support(c, r),
                      c->alive.as<uint8_t>(), lo_of(r), hi_of(r), thr, xb, zb, min_rest);
    if (nccl) {
        GC_TRY(allgather_u32(c, xb + (size_t)c->rank * W, xb, (size_t)W));
        GC_TRY(allgather_u32(c, zb + (size_t)c->rank * W, zb, (size_t)W));
        GC_TRY(allreduce_min_u32(c, min_rest, 1));
    }
    GC_LAUNCH(c, k_zero_finish, grid_for(P * W), kThreads, 0, zb, P * W, c->alive.as<uint8_t>(), tau, level, zrem);
    GC_LAUNCH(c, k_bits_to_list, grid_for(P * W), kThreads, 0, xb, P * W, lists[0], counts[0]);
    GC_TRY(record(c, 11));
    GC_TRY(read_small(c, h, counts[0], sizeof(int)));
    GC_TRY(read_small(c, h + 2, zrem, 8));
    GC_TRY(read_small(c, h + 4, min_rest, 4));
    GC_TRY(sync(c));
    c->stats.scan_ms += elapsed(c, 10, 11);
    {
        const int64_t z = *reinterpret_cast<int64_t*>(h + 2);
        *removed += z;
        c->m_alive_h -= z;
    }
    int nf = h[0];
    if (next_thr) {
        const uint32_t mr = static_cast<uint32_t>(h[4]);
        *next_thr = nf > 0 ? 0u : (mr == 0xFFFFFFFFu ? 0u : mr + 1);
    }
    if (nf > 0) GC_TRY(ensure_rows(c));
    if (nccl) return peel_rounds_nccl(c, thr, level, nf, removed, xb, nb);
    // Loopback virtual ranks (one device): every X edge is enumerated once,
    // with its owner's support copy, and decrements land on the survivors'
    // owner copies directly -- the v2 partition without the exchange.
    // Rounds run in device-side batches like the single-rank peeler.
    const int64_t alive0 = c->m_alive_h;
    int cur = 0, batch = c->trace > 1 ? 1 : 2, last_nf = nf;
    unsigned long long done[2] = {0, 0};
    while (nf > 0) {
        GC_TRY(record(c, 8));
        for (int b = 0; b < batch; ++b) {
            const int nxt = cur ^ 1;
            GC_CUDA(c, cudaMemsetAsync(nb, 0, (size_t)P * W * 4, c->stream));
            PolicyPart pol{xb, part_support(c, 0), c->loop_parts > 1 ? m : 0, W * 32, -1, thr, nb, nullptr, nullptr, 0};
            PeelArgs A{lists[cur], 0, counts[cur], c->dag_src.as<int32_t>(), c->dag_col.as<int32_t>(),
                       c->sym_ptr.as<int64_t>(), c->live_len.as<int32_t>(), c->sym_col.as<int32_t>(),
                       c->sym_eid.as<int32_t>(), c->alive.as<uint8_t>()};
            GC_TRY(launch_peel(c, 148 * 8, A, pol, b == 0 ? (int64_t)nf : 0));
            GC_LAUNCH(c, k_finish_round_dev, 148 * 4, kThreads, 0, lists[cur], counts[cur], c->alive.as<uint8_t>(),
                      tau, level, acc);
            std::swap(xb, nb);
            GC_CUDA(c, cudaMemsetAsync(counts[nxt], 0, sizeof(int), c->stream));
            GC_LAUNCH(c, k_bits_to_list, grid_for(P * W), kThreads, 0, xb, P * W, lists[nxt], counts[nxt]);
            cur = nxt;
        }
        GC_TRY(record(c, 9));
        GC_TRY(read_small(c, h, counts[cur], sizeof(int)));
        GC_TRY(read_small(c, h + 2, acc, 16));
        GC_TRY(sync(c));
        c->stats.peel_kernel_ms += elapsed(c, 8, 9);
        memcpy(done, h + 2, 16);
        if (c->trace)
            fprintf(stderr, "peel-trace part level %d batch %d nf %d rounds %llu removed %llu ms %.4f\n", level, batch,
                    nf, done[1], done[0], elapsed(c, 8, 9));
        c->m_alive_h = alive0 - (int64_t)done[0];
        nf = h[0];
        if (nf > 0) GC_TRY(maybe_compact(c));
        if (c->trace < 2) batch = (nf >= kBatchMaxFront || nf > last_nf) ? 1 : std::min(batch * 2, 16);
        last_nf = nf;
    }
    *removed += (int64_t)done[0];
    c->stats.peel_rounds += (int64_t)done[1];
    return GC_OK;
}

static int peel_setup(gc_ctx* c) {
    const int64_t m = c->m;
    c->rows_live = false;
    GC_TRY(ensure(c, c->alive, (size_t)m));
    GC_TRY(ensure(c, c->front_a, (size_t)m * 4));
    GC_TRY(ensure(c, c->front_b, (size_t)m * 4));
    GC_TRY(ensure(c, c->alist, (size_t)m * 4));
    GC_TRY(ensure(c, c->scal, 1024));
    GC_TRY(host_scratch(c, 4096));
    c->m_alive_h = m;
    c->compact_at = m;
    c->alist_n = -1;
    if (m > 0) {
        GC_LAUNCH(c, k_fill_u8, grid_for(m), kThreads, 0, c->alive.as<uint8_t>(), m, (uint8_t)1);
    }
    c->stats.peel_rounds = 0;
    c->stats.compactions = 0;
    c->stats.peel_kernel_ms = c->stats.scan_ms = c->stats.compact_ms = 0;
    c->stats.peel_sum_min = c->stats.peel_decrements = -1;
    if (c->work_stats) {
        GC_TRY(ensure(c, c->vdeg, (size_t)c->n * 4));
        GC_TRY(ensure(c, c->zlist, (size_t)m * 4));
        GC_CUDA(c, cudaMemsetAsync(c->scal.as<char>() + 672, 0, 16, c->stream));
        if (c->n > 0)
            GC_LAUNCH(c, k_vdeg_init, grid_for(c->n), kThreads, 0, c->dag_ptr.as<int64_t>(), c->in_ptr.as<int64_t>(),
                      c->n, c->vdeg.as<int32_t>());
    }
    const int P = peel_parts(c);
    if (P > 0) {
        const int64_t W = part_words(c, P);
        GC_TRY(ensure(c, c->xbits, (size_t)P * W * 4));
        GC_TRY(ensure(c, c->nbits, (size_t)P * W * 4));
        GC_TRY(ensure(c, c->zbits, (size_t)P * W * 4));
        if (c->loop_parts > 1 && m > 0) {
            // every virtual rank starts from the combined exact support
            GC_TRY(ensure(c, c->sup_parts, (size_t)P * m * 4));
            for (int r = 0; r < P; ++r)
                GC_CUDA(c, cudaMemcpyAsync(c->sup_parts.as<uint32_t>() + (size_t)r * m, c->sup.p, (size_t)m * 4,
                                           cudaMemcpyDeviceToDevice, c->stream));
        }
    }
    return GC_OK;
}

static int peel_any(gc_ctx* c, uint32_t thr, int32_t level, int32_t* round, int64_t* removed,
                    uint32_t* next_thr = nullptr) {
    if (next_thr) *next_thr = 0;
    if (peel_parts(c) > 0) return peel_level_part(c, thr, level, removed, next_thr);
    return peel_level(c, thr, level, round, removed, next_thr);
}

// Work stats of the finished peel: Σ min-degree from its accumulator, and
// D = 3T - Σ S(e) over every edge (a frontier edge's S freezes when it joins
// X, a survivor's ends at its support inside the truss; each decrement took
// one unit from 3T).  Not counted by the partitioned peeler (-1).
static int work_collect(gc_ctx* c, bool peeled) {
    if (!c->work_stats) return GC_OK;
    if (!peeled) {
        c->stats.peel_sum_min = c->stats.peel_decrements = 0;
        return GC_OK;
    }
    if (peel_parts(c) > 0) {
        c->stats.peel_sum_min = c->stats.peel_decrements = -1;
        return GC_OK;
    }
    unsigned long long* tot = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 680);
    GC_CUDA(c, cudaMemsetAsync(tot, 0, 8, c->stream));
    if (c->m > 0) GC_LAUNCH(c, k_sum_u32, grid_for(c->m), kThreads, 0, c->sup.as<uint32_t>(), c->m, tot);
    char* h = static_cast<char*>(c->hpin) + 768;
    GC_TRY(read_small(c, h, c->scal.as<char>() + 672, 16));
    GC_TRY(read_small(c, h + 16, support_hits(c), 8));
    GC_TRY(sync(c));
    const uint64_t* v = reinterpret_cast<const uint64_t*>(h);
    c->stats.peel_sum_min = (int64_t)v[0];
    c->stats.peel_decrements = 3 * (int64_t)v[2] - (int64_t)v[1];
    return GC_OK;
}

int ktruss_analysis(gc_ctx* c, int32_t k, uint64_t* triangles, uint32_t* support_out, uint8_t* alive_out,
                    int64_t* m_alive) {
    const int64_t m = c->m;
    GC_TRY(host_scratch(c, 4096));
    GC_TRY(record(c, 0));
    GC_TRY(support_dag(c));                 // cold: support computed inside every call
    {                                       // the support pass found every triangle once
        unsigned long long* hits = support_hits(c);
        // collective on every rank whatever the output pointers (SPMD callers may differ in NULLs)
        if (c->nccl) GC_TRY(allreduce_u64(c, reinterpret_cast<uint64_t*>(hits), 1));
        if (triangles)
            GC_TRY(read_small(c, static_cast<char*>(c->hpin) + 512, hits, 8));
    }
    if (support_out && m > 0) {             // supports before the peel consumes them
        GC_TRY(ensure(c, c->out_tmp, (size_t)m * 4));
        GC_TRY(scatter_canonical_u32(c, c->sup.as<uint32_t>(), c->out_tmp.as<uint32_t>()));
        GC_TRY(copy_out_staged(c, support_out, c->out_tmp.p, (size_t)m * 4));
    }
    GC_TRY(record(c, 2));
    int64_t removed = 0;
    if (k <= 3) {
        // The 2- and 3-trusses need no peel: an edge in no triangle (S = 0)
        // changes no other support when it goes, so the k-truss is
        // {e : S(e) >= k - 2} straight from the support pass (same on every
        // rank: no collective).
        c->stats.peel_rounds = 0;
        GC_TRY(work_collect(c, false));
        if ((alive_out || m_alive) && m > 0) {
            GC_TRY(ensure(c, c->out_tmp2, (size_t)m));
            GC_TRY(ensure(c, c->alive, (size_t)m));
            unsigned long long* kept = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 656);
            GC_CUDA(c, cudaMemsetAsync(kept, 0, 8, c->stream));
            if (support_out) {           // canonical supports at hand: a coalesced pass
                GC_LAUNCH(c, k_mask_from_support, grid_for(m), kThreads, 0, c->out_tmp.as<uint32_t>(), m,
                          (uint32_t)(k - 2), c->out_tmp2.as<uint8_t>(), kept);
            } else {
                GC_LAUNCH(c, k_mask_from_support, grid_for(m), kThreads, 0, c->sup.as<uint32_t>(), m,
                          (uint32_t)(k - 2), c->alive.as<uint8_t>(), kept);
                GC_TRY(scatter_canonical_u8(c, c->alive.as<uint8_t>(), c->out_tmp2.as<uint8_t>()));
            }
            if (alive_out) GC_TRY(copy_out_staged(c, alive_out, c->out_tmp2.p, (size_t)m));
            GC_TRY(read_small(c, static_cast<char*>(c->hpin) + 520, kept, 8));
            GC_TRY(sync(c));
            removed = m - (int64_t)*reinterpret_cast<uint64_t*>(static_cast<char*>(c->hpin) + 520);
        }
    } else if (alive_out || m_alive || c->nccl) {   // the peel is collective under a communicator
        GC_TRY(peel_setup(c));
        if (m > 0 && k > 2) {
            int32_t round = 0;
            GC_TRY(peel_any(c, (uint32_t)(k - 2), -1, &round, &removed));
        }
        GC_TRY(work_collect(c, m > 0 && k > 2));
        if (alive_out && m > 0) {
            GC_TRY(ensure(c, c->out_tmp2, (size_t)m));
            if (support_out && c->stats.peel_rounds == 0) {
                // no round ran: only zero-support edges left, read the mask off the
                // canonical supports (coalesced) instead of scattering the DAG-order one
                unsigned long long* kept = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 656);
                GC_LAUNCH(c, k_mask_from_support, grid_for(m), kThreads, 0, c->out_tmp.as<uint32_t>(), m, 1u,
                          c->out_tmp2.as<uint8_t>(), kept);
            } else {
                GC_TRY(scatter_canonical_u8(c, c->alive.as<uint8_t>(), c->out_tmp2.as<uint8_t>()));
            }
            GC_TRY(copy_out_staged(c, alive_out, c->out_tmp2.p, (size_t)m));
        }
    }
    GC_TRY(record(c, 1));
    GC_TRY(sync(c));
    if (triangles) *triangles = *reinterpret_cast<uint64_t*>(static_cast<char*>(c->hpin) + 512);
    if (m_alive) *m_alive = m - removed;
    c->stats.ktruss_ms = elapsed(c, 0, 1);
    c->stats.peel_ms = elapsed(c, 2, 1);
    c->stats.support_kernel_ms = elapsed(c, 6, 7);
    return GC_OK;
}

int ktruss(gc_ctx* c, int32_t k, uint8_t* alive_out, int64_t* m_alive) {
    return ktruss_analysis(c, k, nullptr, nullptr, alive_out, m_alive);
}

int truss_decomposition(gc_ctx* c, int32_t* tau_out, int32_t* kmax) {
    const int64_t m = c->m;
    struct DecompFlag {
        gc_ctx* c;
        ~DecompFlag() { c->decomp_running = false; }
    } flag{c};
    c->decomp_running = true;
    GC_TRY(record(c, 0));
    GC_TRY(support_dag(c));
    GC_TRY(record(c, 2));
    GC_TRY(peel_setup(c));
    GC_TRY(ensure(c, c->tau, (size_t)m * 4));
    if (m > 0) GC_LAUNCH(c, k_fill_i32, grid_for(m), kThreads, 0, c->tau.as<int32_t>(), m, (int32_t)2);
    int64_t left = m;
    int32_t last = 0;
    int32_t round = 0;
    for (int32_t k = 3; left > 0; ++k) {
        int64_t removed = 0;
        uint32_t next_thr = 0;
        GC_TRY(peel_any(c, (uint32_t)(k - 2), k - 1, &round, &removed, &next_thr));
        if (removed > 0) last = k - 1;
        left -= removed;
        // skip the levels whose frontier is known to be empty (their k-trusses
        // equal the current one: no trussness value to assign)
        if (next_thr > (uint32_t)(k - 1)) k = (int32_t)next_thr + 1;
    }
    GC_TRY(work_collect(c, m > 0));
    *kmax = (m > 0) ? last : 0;
    GC_TRY(ensure(c, c->out_tmp, (size_t)m * 4));
    if (m > 0)
        GC_TRY(scatter_canonical_u32(c, c->tau.as<uint32_t>(), c->out_tmp.as<uint32_t>()));   // tau >= 2
    GC_TRY(record(c, 1));
    GC_TRY(copy_out(c, tau_out, c->out_tmp.p, (size_t)m * 4));
    GC_TRY(sync(c));
    c->stats.decomp_ms = elapsed(c, 0, 1);
    c->stats.peel_ms = elapsed(c, 2, 1);
    return GC_OK;
}

}  // namespace gcx
