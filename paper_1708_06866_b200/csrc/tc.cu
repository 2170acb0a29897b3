// tc.cu — per-edge triangle support and triangle count (SURVEY §8(a) rows
// a5-a7): work estimate + task binning, and the sm_100a intersection kernels.
//
// Method (P:157-243 [Triangle counting], P:283-288 [k-Truss]): support(u,v) =
// |N(u) ∩ N(v)|; the triangle count is Σ support / 3.  Here every triangle
// is found exactly once in the rank-oriented DAG (Alg. 3's L·U masked by A,
// P:230-243, after relabelling by (degree, id)): for ranks u < v < w the
// triangle is found at its middle vertex v, by its lowest vertex u:
//
//   for each v with d+(v) > 0:  H = hash of N+(v) in shared memory
//     for each in-edge u -> v:  for each w in N+(u) after v (the suffix):
//        w ∈ H  <=>  triangle {u, v, w}
//
// Only the suffix of N+(u) past v can meet N+(v) (its entries all rank
// above v), so the streamed volume is Σ_x C(d+(x), 2) wedges instead of the
// full Σ d-·d+ (DESIGN.md "Kernels").  Per-edge support credits the three
// edges of each triangle found:  (u,v) by a warp reduction over the in-edge's
// hits (one atomic per segment), (v,w) by a shared counter per element of
// N+(v) flushed once per head, (u,w) by one global atomic.
//
// Task classes by d+(v): 0 warp task, 64-slot hash; 1 warp task,
// 512-slot hash; 2 block task, rank-window bitmap (or a 4096-slot hash);
// 3 block task, 16384-slot hash (binary search of N+(v) in global memory only
// past GC_OPT_HUGE_MAX).  Tasks are (v, in-edge range) cut by an exclusive
// scan of a per-in-edge cost so every task holds about task_chunk wedges (8x
// for block tasks); the same cut points give the multi-GPU 1D partition
// (SURVEY §8(e)).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>

#include "gc_internal.cuh"

namespace gcx {

namespace {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
#ifndef GC_KOVH
#define GC_KOVH 128
#endif
#ifndef GC_UW16
#define GC_UW16 1          // (u,w) credits into a separate uint16[m] array (folded into the supports after the
                           // pass): four adjacent positions per 64-bit atomic, half the L2 footprint of the
                           // scattered role.  A count never exceeds d+(u) <= sqrt(2m) < 2^16 (m < 2^31), so
                           // the 16-bit lanes never carry.  0: 32-bit credits straight into the supports
#endif
#ifndef GC_PAIR_CREDIT
#define GC_PAIR_CREDIT 1   // (u,w) credits of adjacent positions paired into 64-bit atomics (C4 / C5 support
                           // pass 99.8 -> 95.3 / 1,282 -> 1,122 ms); 0: one 32-bit atomic per credit
#endif
constexpr int kOvh = GC_KOVH;               // per in-edge overhead in the cost model (cost units)
#ifndef GC_BULK_PF
#define GC_BULK_PF 0       // TMA bulk L2 prefetch (cp.async.bulk.prefetch.L2), bit mask: 1 = each long suffix
                           // whole when the warp starts it, plus the next long one; 2 = every short suffix of a
                           // 32-in-edge group (per-lane addresses: a uniform-register loop); 4 = the next group's
                           // in-edge records (in_pos, in_src, in_cost)
#endif
#ifndef GC_KD1
#define GC_KD1 128
#endif
constexpr int kD0 = 8, kD1 = GC_KD1, kD2 = 4096;    // class bounds on d+(v)
constexpr int kD4 = 8192;                           // class 4 (wide bitmap): d+ bound
constexpr int pow2_at_least(int x) { return x <= 1 ? 1 : 2 * pow2_at_least((x + 1) / 2); }
constexpr int kTS1 = pow2_at_least(2 * kD1);   // class-1 warp hash slots: load <= 1/2 at d+ = kD1
static_assert((kTS1 & (kTS1 - 1)) == 0 && kTS1 >= 2 * kD1, "class-1 table: power of two, load <= 1/2");
constexpr int64_t kTinyChunk = 1024;  // class-0 task budget (cost units): one task per lane, keep lanes even
#ifndef GC_TINY_IN
#define GC_TINY_IN 64
#endif
constexpr int64_t kTinyIn = GC_TINY_IN;   // class 0 also needs at most this many in-edges
constexpr int kBW = 8192;      // heavy-head bitmap words (32 KB); the last one is a zero
constexpr int kBWS = kBW;      // sentinel, so heads spanning <= 32*(kBW-1) ranks fit

extern __shared__ uint32_t g_dsmem[];   // dynamic shared memory of every kernel here
constexpr int kTS2 = 4096;     // heavy-head hash slots when the bitmap does not fit
constexpr int kTS3 = 16384;    // huge-head hash slots (d+ <= kTS3/2 by default)
constexpr int kD2H = 2048;     // largest d+ the heavy-head hash takes (load <= 1/2)
constexpr int kWarps = 8;                   // 256 threads per block
#ifndef GC_SUP_WARPS
#define GC_SUP_WARPS 16                     // heavy-head support kernel: warps per block sharing one table
                                            // (4 x 16 = the SM's 64 warps at 32 registers, a 72-byte spill:
                                            // C4 110.2 -> 102.0 ms against 10 warps at 48 registers; the
                                            // kernel is latency-bound, so occupancy beats the spill)
#endif
#ifndef GC_SUP_MINB
#define GC_SUP_MINB 4                       // ... and resident blocks per SM (register budget)
#endif
#ifndef GC_HUGE_WARPS_TC
#define GC_HUGE_WARPS_TC 20                 // huge-head kernels (class 3): warps per block sharing the
#endif                                      // table (1-3 resident blocks per SM: more warps hide latency)
#ifndef GC_HUGE_WARPS_SUP
#define GC_HUGE_WARPS_SUP 32
#endif
#define GC_HUGE_WARPS(S) ((S) ? GC_HUGE_WARPS_SUP : GC_HUGE_WARPS_TC)
#ifndef GC_HUGE_MINB_TC
#define GC_HUGE_MINB_TC 3                   // huge-head count kernel: resident blocks per SM to budget for (3 x 20 warps at
                                            // 32 registers: C5 TC 520 -> 481 ms against 2 x 16 at 61)
#endif
#ifndef GC_TC_WARPS
#define GC_TC_WARPS 12                      // heavy-head count kernel: warps per block (5 x 12 = 60 warps
                                            // at 32 registers: C4 51.0 -> 49.2 ms, C5 545 -> 523 ms)
#endif
#ifndef GC_WARP_MINB
#define GC_WARP_MINB 8                      // warp-task kernel (class 1): resident blocks per SM to budget for
                                            // (8: 32 registers, 64 warps; C4 support -2 % next to the block kernel)
#endif
#ifndef GC_TINY_MINB
#define GC_TINY_MINB 8                      // lane-task kernel (class 0)
#endif
#ifndef GC_TC_MINB
#define GC_TC_MINB 5
#endif
#ifndef GC_WIDE_MINB
#define GC_WIDE_MINB 3                      // class-4 support kernel (72 KB of shared memory: 3 blocks per SM)
#endif

// Kernel class of head v: 0/1 warp tasks (hash of N+(v) per warp), 2 block
// tasks (rank-window bitmap if N+(v) spans <= bm_bits ranks, else hash when
// d+ <= kD2H), 3 block tasks on a 16384-slot shared hash (one or two blocks
// per SM; d+ above the huge-hash limit searches N+(v) in global memory).
// force raises the class (testing).
__device__ __forceinline__ int head_class(const int64_t* __restrict__ dag_ptr, const int32_t* __restrict__ dag_col,
                                          const int64_t* __restrict__ in_ptr, int v, int force, uint32_t bm_bits) {
    const int64_t r0 = dag_ptr[v];
    const int64_t d = dag_ptr[v + 1] - r0;
    // lane tasks only for tiny heads with few in-edges: a hub with a short
    // N+(v) but many in-neighbours would serialise long suffixes in lanes
    // and pile its (v,w) credits on a handful of global counters
    const bool tiny = d <= kD0 && in_ptr[v + 1] - in_ptr[v] <= kTinyIn;
    int c = tiny ? 0 : d <= kD1 ? 1 : 2;
    if (c < force) c = force;
    if (c == 2) {
        const uint32_t span = d > 0 ? (uint32_t)dag_col[r0 + d - 1] - (uint32_t)v : 0u;
        if (d > kD2 || (span > bm_bits && d > kD2H)) c = 3;
        // class 4: too many (v,w) counters for the block kernel's 4096, but the
        // rank window still holds N+(v): the bitmap kernel with 8192 counters
        // (C5: every head of class 3 -- 7,614 heads, 22 % of the wedges)
        if (c == 3 && force != 3 && d <= kD4 && span <= bm_bits) c = 4;
    }
    return c;
}

__device__ __forceinline__ uint32_t hash_slot(uint32_t w, int lg) { return (w * 0x9E3779B1u) >> (32 - lg); }

__device__ __forceinline__ int table_lg(int d, int max_lg) {
    int lg = 5;                                 // >= 32 slots, load factor <= 1/2
    while ((1 << lg) < 2 * d && lg < max_lg) ++lg;
    return lg;
}

// ------------------------------------------------------------ task build --
__global__ void k_in_cost(const int32_t* __restrict__ in_pos, const int32_t* __restrict__ in_src,
                          const int32_t* __restrict__ in_dst, const int64_t* __restrict__ dag_ptr, int64_t m,
                          int64_t* __restrict__ cost) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m; i += (int64_t)gridDim.x * blockDim.x) {
        if (i == m) { cost[i] = 0; continue; }
        int v = in_dst[i];
        int64_t dv = dag_ptr[v + 1] - dag_ptr[v];
        int64_t len = dag_ptr[in_src[i] + 1] - (int64_t)in_pos[i] - 1;
        cost[i] = (dv > 0 && len > 0) ? len + kOvh : 0;
    }
}

// Per head v: the cost budget of its tasks (0 when v has no work): 8x the
// chunk for block classes, the tiny budget for lane tasks.
__global__ void k_head_chunk(const int64_t* __restrict__ pref, const int64_t* __restrict__ in_ptr,
                             const int64_t* __restrict__ dag_ptr, const int32_t* __restrict__ dag_col, int64_t n,
                             int64_t chunk, int force, uint32_t bm_bits, int64_t* __restrict__ hch) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        int64_t ch = 0;
        if (dag_ptr[v + 1] > dag_ptr[v] && pref[in_ptr[v + 1]] > pref[in_ptr[v]]) {
            const int cl = head_class(dag_ptr, dag_col, in_ptr, (int)v, force, bm_bits);
            ch = cl >= 2 ? chunk * kWarps : cl == 0 ? min(chunk, kTinyChunk) : chunk;   // 2, 3, 4: block tasks
        }
        hch[v] = ch;
    }
}

// floor(x / d) for x >= 0, d > 0: a double quotient corrected in integers
// (exact; one step either way while x < 2^53 -- the total cost is below
// m * sqrt(2m) < 2^48 -- against the int64 division's long software sequence)
__device__ __forceinline__ int64_t floor_div(int64_t x, int64_t d) {
    int64_t q = (int64_t)((double)x / (double)d);
    while (q * d > x) --q;
    while ((q + 1) * d <= x) ++q;
    return q;
}

// A task starts at the first in-edge of every head v that has work, and
// wherever the running cost crosses a multiple of the head's budget or an
// owner boundary (multi-GPU cut).  Zero-cost in-edges (empty suffix) stay
// inside the surrounding task.
__global__ void k_task_flags(const int64_t* __restrict__ pref, const int32_t* __restrict__ in_dst,
                             const int64_t* __restrict__ in_ptr, const int64_t* __restrict__ hch, int64_t m,
                             int64_t total, int parts, uint8_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int v = in_dst[i];
        const int64_t ch = hch[v];
        uint8_t f = 0;
        if (ch > 0) {
            if (i == in_ptr[v]) f = 1;
            else if (floor_div(pref[i], ch) * ch > pref[i - 1]) f = 1;   // a multiple of ch in (pref[i-1], pref[i]]
            else if (parts > 1 && (pref[i] * parts) / total != (pref[i - 1] * parts) / total) f = 1;
        }
        flag[i] = f;
    }
}

__global__ void k_task_cost(const uint64_t* __restrict__ packed, int64_t nt, const int64_t* __restrict__ in_cost,
                            int64_t* __restrict__ cost) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= nt; t += (int64_t)gridDim.x * blockDim.x) {
        if (t == nt) { cost[t] = 0; continue; }
        const uint64_t pk = packed[t];
        cost[t] = in_cost[(uint32_t)(pk >> 32)] - in_cost[(uint32_t)pk];
    }
}

__global__ void k_task_fill(const int32_t* __restrict__ sel, int64_t ntask, int64_t m,
                            const int32_t* __restrict__ in_dst, const int64_t* __restrict__ in_ptr,
                            const int64_t* __restrict__ dag_ptr, const int32_t* __restrict__ dag_col, int force,
                            uint32_t bm_bits, uint32_t* __restrict__ cls, uint64_t* __restrict__ packed,
                            unsigned long long* __restrict__ hist) {
    __shared__ unsigned int bh[kClasses];          // per-block class histogram (one global atomic per class)
    if (threadIdx.x < kClasses) bh[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < ntask; j += (int64_t)gridDim.x * blockDim.x) {
        int i0 = sel[j];
        int v = in_dst[i0];
        int64_t nxt = (j + 1 < ntask) ? (int64_t)sel[j + 1] : m;
        int64_t i1 = min(nxt, in_ptr[v + 1]);
        int k = head_class(dag_ptr, dag_col, in_ptr, v, force, bm_bits);
        cls[j] = (uint32_t)k;
        packed[j] = (uint64_t)(uint32_t)i0 | ((uint64_t)(uint32_t)i1 << 32);
        const unsigned grp = __match_any_sync(__activemask(), k);    // lanes of one class: one shared atomic
        if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(bh + k, (unsigned)__popc(grp));
    }
    __syncthreads();
    if (threadIdx.x < kClasses && bh[threadIdx.x]) atomicAdd(hist + threadIdx.x, (unsigned long long)bh[threadIdx.x]);
}

// roles (u,w) and (u,v) of DAG position q (an edge u -> x): into the uint16
// array (the 32-bit word holding it) or straight into the supports.  The two
// roles count disjoint parts of N+(u) \ {x} -- third vertices below x, and
// above x -- so their sum is below d+(u) <= sqrt(2m) < 2^16: no lane carries.
__device__ __forceinline__ void credit_u(uint32_t* __restrict__ sup, uint16_t* __restrict__ uw16, int64_t q,
                                         uint32_t k) {
#if GC_UW16
    (void)sup;
    atomicAdd(reinterpret_cast<unsigned*>(uw16 + (q & ~(int64_t)1)), k << ((unsigned)(q & 1) << 4));
#else
    (void)uw16;
    atomicAdd(sup + q, k);
#endif
}
__device__ __forceinline__ void credit_uw(uint32_t* __restrict__ sup, uint16_t* __restrict__ uw16, int64_t q) {
    credit_u(sup, uw16, q, 1u);
}

#if GC_BULK_PF
// TMA bulk prefetch of dag_col[beg, beg + len) into L2 (16-byte aligned
// superset; dag_col carries 64 bytes of padding past its end).  The operands of
// UBLKPF are uniform registers: call it with warp-uniform arguments, or the
// compiler loops over the lanes' distinct addresses.
__device__ __forceinline__ void bulk_pf(const int32_t* __restrict__ col, int beg, int len) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(col + beg) & ~(uintptr_t)15;
    const uintptr_t z = (reinterpret_cast<uintptr_t>(col + beg + len) + 15) & ~(uintptr_t)15;
    if (z > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(z - a)) : "memory");
}
#endif

// ------------------------------------------------------- stream routine --
// Walk the suffixes of the in-edges [i0, i1), 32 in-edges per group,
// flattening their wedges across the 32 lanes so short and long suffixes
// both use every lane.  With CLIP, only the wedges whose cost units fall in
// [ca, cb) are visited: in-edge i owns cost units [in_cost[i], in_cost[i] +
// kOvh + len) and its wedge j sits at unit in_cost[i] + kOvh + j, so disjoint
// unit ranges split a task's wedges exactly (the block kernel gives each
// warp one eighth).  probe.loc(w) returns a handle (>= 0) when w is in N+(v), else -1;
// probe.credit(handle) adds the (v,w)-role credit.
template <bool SUP, bool CLIP, class Probe>
__device__ __forceinline__ uint32_t stream_task(int i0, int i1, int64_t cbase, int ca, int cb,
                                                const int32_t* __restrict__ in_pos,
                                                const int32_t* __restrict__ in_src,
                                                const int64_t* __restrict__ in_cost,
                                                const int64_t* __restrict__ dag_ptr,
                                                const int32_t* __restrict__ dag_col, uint32_t* __restrict__ sup,
                                                uint16_t* __restrict__ uw16, Probe& probe, int lane, int long_seg,
                                                int uw) {
    uint32_t hits = 0;
    for (int base = i0; base < i1; base += 32) {
        const int i = base + lane;
        const bool valid = i < i1;
#if GC_BULK_PF & 4
        if (lane == 0 && base + 32 < i1) {   // the next group's in-edge records
            const int nb = base + 32, ne = min(i1, base + 64);
            bulk_pf(in_pos, nb, ne - nb);
            bulk_pf(in_src, nb, ne - nb);
            if (CLIP) bulk_pf(reinterpret_cast<const int32_t*>(in_cost), 2 * nb, 2 * (ne - nb));
        }
#endif
        int p = 0, beg = 0, len = 0;
        if (valid) {
            p = __ldg(in_pos + i);
            int u = __ldg(in_src + i);
            beg = p + 1;
            len = (int)(__ldg(dag_ptr + u + 1) - (int64_t)beg);
            if (CLIP) {
                // cost units relative to the task's first in-edge (a task spans < 2^31 units)
                const int w0 = (int)(__ldg(in_cost + i) - cbase) + kOvh;
                int lo = ca - w0, hi = cb - w0;
                lo = lo < 0 ? 0 : (lo > len ? len : lo);
                hi = hi < 0 ? 0 : (hi > len ? len : hi);
                beg += lo;
                len = hi - lo;
            }
        }
#if GC_BULK_PF & 2
        if (len > 0 && len < long_seg) bulk_pf(dag_col, beg, len);
#endif
        // Long suffixes (the bulk of the wedges): one at a time with the whole
        // warp, 16-byte vector loads, no segment search.
        unsigned longs = __ballot_sync(0xffffffffu, len >= long_seg);
#if GC_BULK_PF & 1
        if (longs) {
            const int s0 = __ffs(longs) - 1;
            const int b0 = __shfl_sync(0xffffffffu, beg, s0), l0 = __shfl_sync(0xffffffffu, len, s0);
            if (lane == 0) bulk_pf(dag_col, b0, l0);
        }
#endif
        while (longs) {
            const int s = __ffs(longs) - 1;
            longs &= longs - 1;
            const int b = __shfl_sync(0xffffffffu, beg, s);
            const int e = b + __shfl_sync(0xffffffffu, len, s);
#if GC_BULK_PF & 1
            if (longs) {   // the next long suffix streams into L2 while this one is probed
                const int s1 = __ffs(longs) - 1;
                const int b1 = __shfl_sync(0xffffffffu, beg, s1), l1 = __shfl_sync(0xffffffffu, len, s1);
                if (lane == 0) bulk_pf(dag_col, b1, l1);
            }
#endif
            uint32_t seg_hits = 0;
            auto visit = [&](int q, int w) {
                const uint32_t inr = (uint32_t)(q - b) < (uint32_t)(e - b);
                if (!SUP) {
                    seg_hits += inr & probe.hit((uint32_t)w);     // branch-free for the bitmap
                } else {
                    const int hd = probe.loc((uint32_t)w);        // located once
                    if (inr && hd >= 0) {
                        ++seg_hits;
                        if (!(uw & 2)) probe.credit(hd, sup);     // role (v,w)
                        if (!(uw & 1)) credit_uw(sup, uw16, q);   // role (u,w)
                    }
                }
            };
            // a vector wholly inside [b, e) needs no per-element bounds checks
            auto visit4 = [&](int q0, const int4& V) {
                if (!SUP) {
                    // count: all four probes in every lane, then a mask of the
                    // positions inside [b, e) (no divergent path at the segment ends)
                    const int klo = max(b - q0, 0), khi = min(e - q0, 4);
                    const uint32_t in4 = khi > klo ? (1u << khi) - (1u << klo) : 0u;
                    const uint32_t h4 = probe.hit((uint32_t)V.x) | (probe.hit((uint32_t)V.y) << 1) |
                                        (probe.hit((uint32_t)V.z) << 2) | (probe.hit((uint32_t)V.w) << 3);
                    seg_hits += __popc(h4 & in4);
                } else if (Probe::kBranchFree || GC_PAIR_CREDIT) {
                    // support: the four probes first (independent loads the
                    // compiler cannot move past the credits' shared atomics,
                    // which might alias), then the hits
                    const int h0 = probe.loc((uint32_t)V.x), h1 = probe.loc((uint32_t)V.y),
                              h2 = probe.loc((uint32_t)V.z), h3 = probe.loc((uint32_t)V.w);
#if GC_PAIR_CREDIT
                    // role (u,w) of two adjacent positions in one 64-bit atomic:
                    // q0 is a multiple of 4, so (q0, q0+1) and (q0+2, q0+3) are
                    // aligned u32 pairs, and a count never carries into its
                    // neighbour (supports stay below 2^31)
                    auto hit = [&](int q, int hd) -> uint32_t {
                        return ((uint32_t)(q - b) < (uint32_t)(e - b) && hd >= 0) ? 1u : 0u;
                    };
                    const uint32_t k0 = hit(q0, h0), k1 = hit(q0 + 1, h1), k2 = hit(q0 + 2, h2), k3 = hit(q0 + 3, h3);
                    seg_hits += k0 + k1 + k2 + k3;
                    if (!(uw & 2)) {                                     // role (v,w)
                        if (k0) probe.credit(h0, sup);
                        if (k1) probe.credit(h1, sup);
                        if (k2) probe.credit(h2, sup);
                        if (k3) probe.credit(h3, sup);
                    }
                    if (!(uw & 1)) {
#if GC_UW16
                        // the four positions q0..q0+3 (q0 a multiple of 4): one 64-bit atomic
                        if (k0 | k1 | k2 | k3)
                            atomicAdd(reinterpret_cast<unsigned long long*>(uw16 + q0),
                                      (unsigned long long)k0 | ((unsigned long long)k1 << 16) |
                                          ((unsigned long long)k2 << 32) | ((unsigned long long)k3 << 48));
#else
                        if (k0 | k1)
                            atomicAdd(reinterpret_cast<unsigned long long*>(sup + q0),
                                      ((unsigned long long)k1 << 32) | k0);
                        if (k2 | k3)
                            atomicAdd(reinterpret_cast<unsigned long long*>(sup + q0 + 2),
                                      ((unsigned long long)k3 << 32) | k2);
#endif
                    }
#else
                    auto take = [&](int q, int hd) {
                        if ((uint32_t)(q - b) < (uint32_t)(e - b) && hd >= 0) {
                            ++seg_hits;
                            if (!(uw & 2)) probe.credit(hd, sup);     // role (v,w)
                            if (!(uw & 1)) credit_uw(sup, uw16, q);   // role (u,w)
                        }
                    };
                    take(q0, h0); take(q0 + 1, h1); take(q0 + 2, h2); take(q0 + 3, h3);
#endif
                } else {
                    visit(q0, V.x); visit(q0 + 1, V.y); visit(q0 + 2, V.z); visit(q0 + 3, V.w);
                }
            };
            // two 16-byte loads in flight per lane (256 wedges per warp step)
            for (int q0 = (b & ~3) + lane * 4; q0 < e; q0 += 256) {
                const int4 A = __ldg(reinterpret_cast<const int4*>(dag_col + q0));
                const bool two = q0 + 128 < e;
                int4 B = make_int4(0, 0, 0, 0);
                if (two) B = __ldg(reinterpret_cast<const int4*>(dag_col + q0 + 128));
                visit4(q0, A);
                if (two) visit4(q0 + 128, B);
            }
            hits += seg_hits;
            if (SUP) {
                const uint32_t tot_hits = __reduce_add_sync(0xffffffffu, seg_hits);
                const int ps = __shfl_sync(0xffffffffu, p, s);
                if (lane == 0 && tot_hits && !(uw & 4)) credit_u(sup, uw16, ps, tot_hits);   // role (u,v)
            }
        }
        if (len >= long_seg) len = 0;
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        const int excl = incl - len;
        for (int k = 0; k < tot; k += 32) {
            const int t = k + lane;
            int s = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                int e = __shfl_sync(0xffffffffu, excl, s + step);
                if (e <= t) s += step;
            }
            const int es = __shfl_sync(0xffffffffu, excl, s);
            const int bs = __shfl_sync(0xffffffffu, beg, s);
            const int ps = SUP ? __shfl_sync(0xffffffffu, p, s) : 0;
            bool hit = false;
            if (t < tot) {
                const int q = bs + (t - es);
                const uint32_t w = (uint32_t)__ldg(dag_col + q);
                if (!SUP) {
                    hits += probe.hit(w);
                } else {
                    const int slot = probe.loc(w);
                    if (slot >= 0) {
                        hit = true;
                        ++hits;
                        if (!(uw & 2)) probe.credit(slot, sup);   // role (v,w)
                        if (!(uw & 1)) credit_uw(sup, uw16, q);   // role (u,w)
                    }
                }
            }
            if (SUP) {
                // role (u,v): lanes of one segment are contiguous; one atomic per segment
                const unsigned hm = __ballot_sync(0xffffffffu, hit);
                if (hit && !(uw & 4)) {
                    const unsigned grp = __match_any_sync(hm, s);
                    if (lane == __ffs(grp) - 1) credit_u(sup, uw16, ps, (uint32_t)__popc(grp));
                }
            }
        }
    }
    return hits;
}

// Shared-memory open-addressing table of N+(v): keys = rank ids, vals =
// index j within N+(v), cnt = (v,w)-role credits.
template <bool SUP>
struct SmemHash {
    static constexpr bool kBranchFree = false;
    uint32_t* keys;
    int32_t* vals;
    uint32_t* cnt;
    int lg;
    uint32_t mask;
    __device__ __forceinline__ int find(uint32_t w) const {
        uint32_t h = hash_slot(w, lg);
        while (true) {
            uint32_t k = keys[h];
            if (k == w) return (int)h;
            if (k == kEmpty) return -1;
            h = (h + 1) & mask;
        }
    }
    __device__ __forceinline__ int loc(uint32_t w) const { return find(w); }
    __device__ __forceinline__ void credit(int slot, uint32_t*) const {
        if (SUP) atomicAdd(cnt + slot, 1u);
    }
    __device__ __forceinline__ uint32_t hit(uint32_t w) const { return find(w) >= 0; }
};

#ifndef GC_DYN_BATCH
#define GC_DYN_BATCH 1   // block classes fetch batches from a global counter (0: static round-robin)
#endif

struct KArgs {
    const int32_t* in_pos;
    const int32_t* in_src;
    const int32_t* in_dst;
    const int64_t* in_cost;
    const int64_t* dag_ptr;
    const int32_t* dag_col;
    const uint64_t* tasks;      // packed (i0, i1), this class's slice
    int64_t ntask;
    int64_t total_cost;
    int parts, owner;           // skip tasks not owned by `owner` of `parts`
    const int64_t* task_pref;   // exclusive cost prefix over the tasks (this class's slice)
    int64_t cls_start, cls_total;   // ... the class's first prefix value and its total cost
    uint32_t* sup;
    uint16_t* uw16;             // (u,w)-role credits (GC_UW16), folded into sup after the pass
    unsigned long long* count;
    uint32_t bm_bits;           // bitmap capacity of the heavy-head kernel (0: hash only)
    int long_seg;               // suffix length threshold of the warp-vector path
    int batch;                  // heavy-head kernel: consecutive tasks per batch
    int uw;                     // diagnostics: support roles skipped (GC_OPT_SUP_SKIP mask)
    int huge_max;               // class 3: largest d+ held in the shared hash
    unsigned long long* next;   // block classes: batch counter (zeroed per launch; null: static dealing)
    long long* slot;            // ... and 2 slots per block publishing the next batch id to its warps
};

// 1D cut per class: task t of a class belongs to owner
// floor((cost of the class's tasks before t) * parts / class total), so every
// owner gets 1/parts of every class's cost units.  (One cut over all classes
// gave the owner of the lowest-ranked heads -- warp and lane tasks, dearer per
// cost unit than block tasks -- 1.9x the mean TC time at 8 loopback parts.)
__device__ __forceinline__ bool owned(const KArgs& a, int64_t t) {
    if (a.parts <= 1) return true;
    return (int)(((a.task_pref[t] - a.cls_start) * a.parts) / a.cls_total) == a.owner;
}

__device__ __forceinline__ void add_count(unsigned long long* count, uint32_t hits, int lane) {
    unsigned long long h = hits;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if (lane == 0 && h) atomicAdd(count, h);
}

// ------------------------------------------------ lane-task kernel (0) --
// Tiny heads (d+(v) <= 8), the bulk of the heads of uniform-degree graphs
// (king grids, ER) and of the R-MAT periphery: one task per lane, N+(v) in
// eight registers, each suffix element compared against all of them.  A
// warp thus keeps 32 independent tasks' loads in flight instead of
// building a shared table per head.  Suffix scans stop past max N+(v).
template <bool SUP>
__global__ void __launch_bounds__(256, GC_TINY_MINB) k_tc_tiny(KArgs a) {
    const int lane = threadIdx.x & 31;
    uint32_t hits = 0;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < a.ntask; t += nt) {
        const uint64_t pk = a.tasks[t];
        const int i0 = (int)(uint32_t)pk, i1 = (int)(pk >> 32);
        if (!owned(a, t)) continue;
        const int v = __ldg(a.in_dst + i0);
        const int64_t r0 = __ldg(a.dag_ptr + v);
        const int d = (int)(__ldg(a.dag_ptr + v + 1) - r0);
        int32_t sv[kD0];
#pragma unroll
        for (int k = 0; k < kD0; ++k) sv[k] = k < d ? __ldg(a.dag_col + r0 + k) : -1;
        const int32_t vmax = sv[0] < 0 ? -1 : __ldg(a.dag_col + r0 + d - 1);
        for (int i = i0; i < i1; ++i) {
            const int p = __ldg(a.in_pos + i);
            const int u = __ldg(a.in_src + i);
            const int64_t e = __ldg(a.dag_ptr + u + 1);
            uint32_t seg = 0;
            for (int64_t q = p + 1; q < e; ++q) {
                const int32_t w = __ldg(a.dag_col + q);
                if (w > vmax) break;                       // rows ascend: nothing further can match
                uint32_t mk = 0;
#pragma unroll
                for (int k = 0; k < kD0; ++k) mk |= (uint32_t)(w == sv[k]) << k;
                if (mk) {
                    ++seg;
                    if (SUP) {
                        if (!(a.uw & 1)) credit_uw(a.sup, a.uw16, q);                  // role (u,w)
                        if (!(a.uw & 2)) atomicAdd(a.sup + r0 + (__ffs(mk) - 1), 1u);  // role (v,w)
                    }
                }
            }
            hits += seg;
            if (SUP && seg && !(a.uw & 4)) credit_u(a.sup, a.uw16, p, seg);             // role (u,v)
        }
    }
    add_count(a.count, hits, lane);
}

// ------------------------------------------------- warp-task kernel (1) --
template <int TS, bool SUP>
__global__ void __launch_bounds__(256, GC_WARP_MINB) k_tc_warp(KArgs a) {
    uint32_t* const smem = g_dsmem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int per_warp = SUP ? 3 * TS : TS;
    uint32_t* keys = smem + warp * per_warp;
    int32_t* vals = reinterpret_cast<int32_t*>(keys + TS);
    uint32_t* cnt = keys + 2 * TS;
    constexpr int max_lg = __builtin_ctz(TS);
    uint32_t hits = 0;
    // static round-robin over tasks (every task's cost is bounded by the chunk)
    const int64_t nw = (int64_t)gridDim.x * kWarps;
    for (int64_t t = (int64_t)blockIdx.x * kWarps + warp; t < a.ntask; t += nw) {
        const uint64_t pk = a.tasks[t];
        const int i0 = (int)(uint32_t)pk, i1 = (int)(pk >> 32);
        if (!owned(a, t)) continue;
        const int v = __ldg(a.in_dst + i0);
        const int64_t r0 = __ldg(a.dag_ptr + v);
        const int d = (int)(__ldg(a.dag_ptr + v + 1) - r0);
        const int lg = table_lg(d, max_lg);
        const int ts = 1 << lg;
        for (int j = lane; j < ts; j += 32) {
            keys[j] = kEmpty;
            if (SUP) cnt[j] = 0;
        }
        __syncwarp();
        for (int j = lane; j < d; j += 32) {
            uint32_t w = (uint32_t)__ldg(a.dag_col + r0 + j);
            uint32_t h = hash_slot(w, lg);
            while (atomicCAS(keys + h, kEmpty, w) != kEmpty) h = (h + 1) & (ts - 1);
            if (SUP) vals[h] = j;
        }
        __syncwarp();
        SmemHash<SUP> H{keys, vals, cnt, lg, (uint32_t)(ts - 1)};
        hits += stream_task<SUP, false>(i0, i1, 0, 0, 0, a.in_pos, a.in_src, a.in_cost, a.dag_ptr, a.dag_col, a.sup,
                                        a.uw16, H, lane, a.long_seg, a.uw);
        if (SUP) {
            __syncwarp();
            for (int j = lane; j < ts; j += 32)
                if (cnt[j]) atomicAdd(a.sup + r0 + vals[j], cnt[j]);
        }
        __syncwarp();
    }
    add_count(a.count, hits, lane);
}

// ------------------------------------------------- block-task kernel (2) --
// Heavy heads (257 <= d+(v) <= 4096).  N+(v) is held as a bitmap over the
// rank window (v, v + 32*kBW] when its largest element fits (one LDS per
// probe, no probe chains), else as the 8192-slot hash.  The task's wedges
// are split exactly into 8 equal cost-unit slices, one per warp, so the
// block barrier after the stream does not wait on a straggler warp.

template <bool SUP>
struct SmemBitmap {
    static constexpr bool kBranchFree = true;   // loc() is one LDS, no probe chain
    const uint32_t* bits;    // == g_dsmem (word 0 of the dynamic shared memory)
    const uint16_t* pre;     // SUP: index in N+(v) of the first element of each 64-bit chunk
    uint32_t* cnt;           // SUP: (v,w)-role credits per index j
    uint32_t base;           // v + 1
    // membership only, branch-free: one LDS from the shared window (no
    // generic-pointer conversion).  Words past the head's span are zero and
    // word kBW-1 is a permanent zero sentinel, so clamping the word index is
    // the whole range check (w > v always, so x never wraps).
    __device__ __forceinline__ uint32_t hit(uint32_t w) const {
        const uint32_t x = w - base;
        const uint32_t word = g_dsmem[min(x >> 5, (uint32_t)(kBW - 1))];
        return (word >> (x & 31)) & 1u;
    }
    // handle of a member = its window offset x (branch-free test as in hit())
    __device__ __forceinline__ int loc(uint32_t w) const {
        const uint32_t x = w - base;
        const uint32_t word = g_dsmem[min(x >> 5, (uint32_t)(kBW - 1))];
        return ((word >> (x & 31)) & 1u) ? (int)x : -1;
    }
    // role (v,w): the index j of w in N+(v) = set bits before x; pre holds the
    // index of the first element of each 64-bit chunk
    __device__ __forceinline__ void credit(int hd, uint32_t*) const {
        if (!SUP) return;
        const uint32_t x = (uint32_t)hd;
        const uint64_t chunk = reinterpret_cast<const uint64_t*>(bits)[x >> 6];   // one 64-bit LDS
        const int j = (int)pre[x >> 6] + __popcll(chunk & ((1ull << (x & 63)) - 1ull));
        atomicAdd(cnt + j, 1u);
    }
};

// Smallest i in [lo, hi) with a[i] >= x (hi if none); one warp, 32-ary search.
__device__ __forceinline__ int64_t warp_lower_bound(const int64_t* __restrict__ a, int64_t lo, int64_t hi, int64_t x,
                                                    int lane) {
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t pos = lo + lane * step;
        const bool less = pos < hi && __ldg(a + pos) < x;
        const int c = __popc(__ballot_sync(0xffffffffu, less));
        const int64_t nlo = c > 0 ? lo + (int64_t)(c - 1) * step + 1 : lo;
        const int64_t nhi = c < 32 ? min(hi, lo + (int64_t)c * step) : hi;
        lo = nlo;
        hi = nhi;
    }
    const int64_t pos = lo + lane;
    const bool less = pos < hi && __ldg(a + pos) < x;
    return lo + __popc(__ballot_sync(0xffffffffu, less));
}

// Probe of N+(v) in global memory (binary search): huge heads past the table.
struct GlobalProbe {
    static constexpr bool kBranchFree = false;
    const int32_t* row;
    int d;
    int64_t r0;
    __device__ __forceinline__ int find(uint32_t w) const {
        int lo = 0, hi = d;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if ((uint32_t)__ldg(row + mid) < w) lo = mid + 1; else hi = mid;
        }
        return (lo < d && (uint32_t)__ldg(row + lo) == w) ? lo : -1;
    }
    __device__ __forceinline__ int loc(uint32_t w) const { return find(w); }
    __device__ __forceinline__ void credit(int j, uint32_t* sup) const { atomicAdd(sup + r0 + j, 1u); }
    __device__ __forceinline__ uint32_t hit(uint32_t w) const { return find(w) >= 0; }
};

template <bool SUP, bool HUGE, int KD = kD2>   // KD: bitmap-mode (v,w) counters (kD4 for class 4)
__global__ void __launch_bounds__(32 * (HUGE ? GC_HUGE_WARPS(SUP) : SUP ? GC_SUP_WARPS : GC_TC_WARPS),
                                  HUGE ? (SUP ? 1 : GC_HUGE_MINB_TC)
                                       : (SUP ? (KD > kD2 ? GC_WIDE_MINB : GC_SUP_MINB) : GC_TC_MINB))
    k_tc_block(KArgs a) {
    constexpr int BW = HUGE ? GC_HUGE_WARPS(SUP) : SUP ? GC_SUP_WARPS : GC_TC_WARPS;   // warps per block (= blockDim.x / 32)
    uint32_t* const smem = g_dsmem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // layout (32-bit words): [0, kBW) bitmap | hash keys+vals ;
    // SUP: [kBW, kBW + kBW/4) u16 prefix per 64-bit chunk | hash cnt ; then KD bitmap-mode cnt
    // HUGE (class 3): [0, kTS3) keys | [kTS3, 2 kTS3) vals | [2 kTS3, 3 kTS3) cnt (SUP only)
    constexpr int kTSH = HUGE ? kTS3 : kTS2;
    constexpr int kZero = HUGE ? kTS3 : kBWS;    // words kept zero between heads
    uint32_t* bits = smem;
    uint32_t* keys = smem;
    int32_t* vals = reinterpret_cast<int32_t*>(smem + kTSH);
    uint16_t* pre = reinterpret_cast<uint16_t*>(smem + kBWS);    // kBW/2 u16 = kBW/4 words
    uint32_t* hcnt = HUGE ? smem + 2 * kTS3 : smem + kBWS;        // hash mode: kTSH words
    uint32_t* bcnt = smem + kBWS + kBW / 4;                        // bitmap mode: KD words
    static_assert(kTS2 <= kBW / 4 + kD2, "hash counters fit the SUP region");
    constexpr int max_lg = __builtin_ctz(kTSH);
    static_assert(2 * kTS2 <= kBW && kTS2 <= kBW / 2, "hash fits the bitmap region");
    uint32_t hits = 0;
    // Tasks are dealt to blocks in batches of a.batch consecutive tasks,
    // round-robin, so all blocks advance through the heads in rank order
    // together (adjacent hubs share in-neighbours, whose rows then hit in L2)
    // while consecutive tasks of one head share its table: the block
    // synchronises only when the head changes.  Invariant: the bitmap region
    // is all zero between heads.
    const int64_t nbatch = (a.ntask + a.batch - 1) / a.batch;
    // the next batch id goes through global memory (a per-block slot pair):
    // 16 more bytes of static shared memory would cost the support kernel a
    // resident block per SM (4 x 57,344 B + reserve fill the SM exactly)
    long long* s_bt = a.slot + 2 * blockIdx.x;
    if (threadIdx.x == 0) s_bt[0] = blockIdx.x;
    for (int j = threadIdx.x; j < kZero; j += blockDim.x) bits[j] = 0u;
    int cur = -1, d = 0, lg = 0, ts = 0;
    int64_t r0 = 0;
    uint32_t span = 0;
    bool use_bm = false, use_gp = false;   // use_gp: N+(v) too large for the table, search it in global memory
    auto teardown = [&](bool clear) {
        if (SUP && !use_gp) {
            if (use_bm) {
                for (int j = threadIdx.x; j < d; j += blockDim.x)
                    if (bcnt[j]) atomicAdd(a.sup + r0 + j, bcnt[j]);
            } else {
                for (int j = threadIdx.x; j < ts; j += blockDim.x)
                    if (hcnt[j]) atomicAdd(a.sup + r0 + vals[j], hcnt[j]);
            }
        }
        if (clear && !use_gp) {
            if (use_bm) {
                for (int j = threadIdx.x; j < d; j += blockDim.x)
                    bits[((uint32_t)__ldg(a.dag_col + r0 + j) - (uint32_t)cur - 1u) >> 5] = 0u;
            } else {
                for (int j = threadIdx.x; j < ts; j += blockDim.x) {
                    keys[j] = 0u;
                    if (!HUGE) vals[j] = 0;   // shares the bitmap region (kept zero); HUGE TC has no vals
                }
            }
        }
    };
    __syncthreads();
    // Batches after the first come from a global counter, in order: blocks
    // stay on neighbouring heads (a static stride lets them drift apart) and
    // no block is left with a long queue at the end.  The next batch id is
    // fetched at the start of a batch into the other slot of s_bt; the
    // barrier closing each batch publishes it.
    for (int par = 0;; par ^= 1) {
    const int64_t bt = *(volatile long long*)(s_bt + par);
    if (bt >= nbatch) break;
    if (threadIdx.x == 0)
        s_bt[par ^ 1] = a.next ? (long long)gridDim.x + (long long)atomicAdd(a.next, 1ull) : bt + gridDim.x;
    for (int64_t t = bt * a.batch; t < min(a.ntask, (bt + 1) * a.batch); ++t) {
        const uint64_t pk = a.tasks[t];
        const int i0 = (int)(uint32_t)pk, i1 = (int)(pk >> 32);
        if (!owned(a, t)) continue;
        const int v = __ldg(a.in_dst + i0);
        if (v != cur) {
            __syncthreads();                      // every warp is done with cur's table
            if (cur >= 0) teardown(true);
            __syncthreads();
            cur = v;
            r0 = __ldg(a.dag_ptr + v);
            d = (int)(__ldg(a.dag_ptr + v + 1) - r0);
            span = (uint32_t)__ldg(a.dag_col + r0 + d - 1) - (uint32_t)v;   // max rank - v
            use_bm = !HUGE && span <= a.bm_bits;
            use_gp = HUGE && d > a.huge_max;
            if (use_gp) {
                // nothing to stage
            } else if (use_bm) {
                for (int j = threadIdx.x; j < d; j += blockDim.x) {
                    if (SUP) bcnt[j] = 0u;
                    const uint32_t x = (uint32_t)__ldg(a.dag_col + r0 + j) - (uint32_t)v - 1u;
                    atomicOr(bits + (x >> 5), 1u << (x & 31));
                    if (SUP) {
                        const bool first = j == 0 ||
                            (((uint32_t)__ldg(a.dag_col + r0 + j - 1) - (uint32_t)v - 1u) >> 6) != (x >> 6);
                        if (first) pre[x >> 6] = (uint16_t)j;
                    }
                }
            } else {
                lg = table_lg(d, max_lg);
                ts = 1 << lg;
                for (int j = threadIdx.x; j < ts; j += blockDim.x) {
                    keys[j] = kEmpty;
                    if (SUP) hcnt[j] = 0;
                }
                __syncthreads();
                for (int j = threadIdx.x; j < d; j += blockDim.x) {
                    uint32_t w = (uint32_t)__ldg(a.dag_col + r0 + j);
                    uint32_t h = hash_slot(w, lg);
                    while (atomicCAS(keys + h, kEmpty, w) != kEmpty) h = (h + 1) & (ts - 1);
                    if (SUP) vals[h] = j;
                }
            }
            __syncthreads();
        }
        // this warp's eighth of the task's cost units
        const int64_t c0 = __ldg(a.in_cost + i0), c1 = __ldg(a.in_cost + i1);
        const int64_t ca = c0 + (c1 - c0) * warp / BW, cb = c0 + (c1 - c0) * (warp + 1) / BW;
        const int ca32 = (int)(ca - c0), cb32 = (int)(cb - c0);
        if (cb > ca) {
            const int first = (int)warp_lower_bound(a.in_cost, i0, i1, ca + 1, lane) - 1;
            const int end = (int)warp_lower_bound(a.in_cost, i0, i1, cb, lane);
            if (use_gp) {
                GlobalProbe G{a.dag_col + r0, d, r0};
                hits += stream_task<SUP, true>(first, end, c0, ca32, cb32, a.in_pos, a.in_src, a.in_cost, a.dag_ptr,
                                               a.dag_col, a.sup, a.uw16, G, lane, a.long_seg, a.uw);
            } else if (use_bm) {
                SmemBitmap<SUP> B{bits, pre, bcnt, (uint32_t)v + 1u};
                hits += stream_task<SUP, true>(first, end, c0, ca32, cb32, a.in_pos, a.in_src, a.in_cost, a.dag_ptr,
                                               a.dag_col, a.sup, a.uw16, B, lane, a.long_seg, a.uw);
            } else {
                SmemHash<SUP> H{keys, vals, hcnt, lg, (uint32_t)(ts - 1)};
                hits += stream_task<SUP, true>(first, end, c0, ca32, cb32, a.in_pos, a.in_src, a.in_cost, a.dag_ptr,
                                               a.dag_col, a.sup, a.uw16, H, lane, a.long_seg, a.uw);
            }
        }
    }
    __syncthreads();
    }
    if (cur >= 0) teardown(false);
    add_count(a.count, hits, lane);
}

// sup[p] += uw16[p], four positions per thread
__global__ void k_fold_uw(uint32_t* __restrict__ sup, const uint16_t* __restrict__ uw16, int64_t m) {
    const int64_t nq = m / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nq; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < nq) {
            uint4 s = reinterpret_cast<uint4*>(sup)[i];
            const uint2 w = reinterpret_cast<const uint2*>(uw16)[i];
            s.x += w.x & 0xFFFFu;
            s.y += w.x >> 16;
            s.z += w.y & 0xFFFFu;
            s.w += w.y >> 16;
            reinterpret_cast<uint4*>(sup)[i] = s;
        } else {
            for (int64_t p = 4 * nq; p < m; ++p) sup[p] += uw16[p];
        }
    }
}

template <class T>
__global__ void k_scatter_t(const T* __restrict__ vals, const int32_t* __restrict__ eid, int64_t m,
                            T* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x)
        out[eid[p]] = vals[p];
}


template <class K>
int occupancy_grid(K kernel, size_t smem, int threads = 256) {
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, threads, smem) != cudaSuccess || blocks < 1) {
        cudaGetLastError();
        blocks = 1;
    }
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return blocks * sms;
}

}  // namespace

static uint32_t bm_bits_of(const gc_ctx* c) { return c->block_bitmap ? (uint32_t)(kBW - 1) * 32u : 0u; }

int prepare_tasks(gc_ctx* c) {
    const int64_t m = c->m;
    c->tasks_ready = false;
    for (int k = 0; k < kClasses; ++k) c->ntask[k] = 0;
    for (int k = 0; k <= kClasses; ++k) c->task_off[k] = 0;
    c->total_cost = 0;
    c->task_parts = c->loop_parts > 0 ? c->loop_parts : c->nranks;
    if (m == 0) {
        c->tasks_ready = true;
        return GC_OK;
    }
    GC_TRY(ensure(c, c->in_cost, (size_t)(m + 1) * 8));
    GC_TRY(ensure(c, c->tmp_a, (size_t)(m + 1) * 8));      // cost, then packed tasks (sorted)
    GC_TRY(ensure(c, c->tmp_b, (size_t)(m + 1) * 8));      // packed tasks (unsorted)
    GC_TRY(ensure(c, c->task_i0, (size_t)(m + 1) * 8));    // final packed tasks
    GC_TRY(ensure(c, c->vals_a, (size_t)(m + 1) * 4));     // flags (uint8) / selected indices
    GC_TRY(ensure(c, c->vals_b, (size_t)(m + 1) * 4));
    GC_TRY(ensure(c, c->keys_a, (size_t)(m + 1) * 8));
    GC_TRY(ensure(c, c->scal, 1024));
    GC_TRY(host_scratch(c, 4096));
    int64_t* h = static_cast<int64_t*>(c->hpin);
    int64_t* cost = c->tmp_a.as<int64_t>();
    GC_LAUNCH(c, k_in_cost, grid_for(m + 1), kThreads, 0, c->in_pos.as<int32_t>(), c->in_src.as<int32_t>(),
              c->in_dst.as<int32_t>(), c->dag_ptr.as<int64_t>(), m, cost);
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, cost, c->in_cost.as<int64_t>(), m + 1, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, cost, c->in_cost.as<int64_t>(), m + 1, c->stream));
    c->stats.lib_launches += 2;
    GC_TRY(read_small(c, h, c->in_cost.as<int64_t>() + m, 8));
    GC_TRY(sync(c));
    c->total_cost = h[0];
    if (c->total_cost == 0) {
        c->tasks_ready = true;
        return GC_OK;
    }
    uint8_t* flags = reinterpret_cast<uint8_t*>(c->vals_b.p);
    GC_TRY(ensure(c, c->keys_b, (size_t)(c->n + 1) * 8));
    int64_t* hch = c->keys_b.as<int64_t>();                 // free after the build
    GC_LAUNCH(c, k_head_chunk, grid_for(c->n), kThreads, 0, c->in_cost.as<int64_t>(), c->in_ptr.as<int64_t>(),
              c->dag_ptr.as<int64_t>(), c->dag_col.as<int32_t>(), c->n, c->task_chunk, c->force_class, bm_bits_of(c),
              hch);
    GC_LAUNCH(c, k_task_flags, grid_for(m), kThreads, 0, c->in_cost.as<int64_t>(), c->in_dst.as<int32_t>(),
              c->in_ptr.as<int64_t>(), hch, m, c->total_cost, 1, flags);
    int32_t* sel = c->vals_a.as<int32_t>();
    int64_t* d_nsel = reinterpret_cast<int64_t*>(c->scal.as<char>() + 128);
    thrust::counting_iterator<int32_t> iota(0);
    tmp = 0;
    GC_CUDA(c, cub::DeviceSelect::Flagged(nullptr, tmp, iota, flags, sel, d_nsel, m, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, iota, flags, sel, d_nsel, m, c->stream));
    c->stats.lib_launches += 2;
    GC_TRY(read_small(c, h, d_nsel, 8));
    GC_TRY(sync(c));
    const int64_t nt = h[0];
    unsigned long long* hist = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 400);   // kClasses
    GC_CUDA(c, cudaMemsetAsync(hist, 0, kClasses * 8, c->stream));
    uint32_t* cls = reinterpret_cast<uint32_t*>(c->keys_a.p);
    uint32_t* cls_sorted = cls + (m + 1);
    GC_LAUNCH(c, k_task_fill, grid_for(nt), kThreads, 0, sel, nt, m, c->in_dst.as<int32_t>(), c->in_ptr.as<int64_t>(),
              c->dag_ptr.as<int64_t>(), c->dag_col.as<int32_t>(), c->force_class, bm_bits_of(c), cls,
              c->tmp_b.as<uint64_t>(), hist);
    tmp = 0;
    GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, cls, cls_sorted, c->tmp_b.as<uint64_t>(),
                                               c->task_i0.as<uint64_t>(), nt, 0, 3, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, cls, cls_sorted, c->tmp_b.as<uint64_t>(),
                                               c->task_i0.as<uint64_t>(), nt, 0, 3, c->stream));
    c->stats.lib_launches += 3;
    GC_TRY(read_small(c, h, hist, kClasses * 8));
    GC_TRY(sync(c));
    int64_t off = 0;
    for (int k = 0; k < kClasses; ++k) {
        c->ntask[k] = h[k];
        c->stats.tasks[k] = h[k];
        c->task_off[k] = off;
        off += h[k];
    }
    c->task_off[kClasses] = off;
    if (c->task_parts > 1 && nt > 0) {
        // per-class 1D cut: exclusive cost prefix over the class-sorted tasks
        GC_TRY(ensure(c, c->task_pref, (size_t)(nt + 1) * 8));
        int64_t* tcost = c->tmp_a.as<int64_t>();           // free after the task build
        GC_LAUNCH(c, k_task_cost, grid_for(nt + 1), kThreads, 0, c->task_i0.as<uint64_t>(), nt,
                  c->in_cost.as<int64_t>(), tcost);
        size_t tmp3 = 0;
        GC_CUDA(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp3, tcost, c->task_pref.as<int64_t>(), nt + 1, c->stream));
        GC_TRY(ensure(c, c->cub_tmp, tmp3));
        tmp3 = c->cub_tmp.cap;
        GC_CUDA(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp3, tcost, c->task_pref.as<int64_t>(), nt + 1,
                                                 c->stream));
        c->stats.lib_launches += 2;
        for (int k = 0; k <= kClasses; ++k)
            GC_TRY(read_small(c, h + 8 + k, c->task_pref.as<int64_t>() + c->task_off[k], 8));
        GC_TRY(sync(c));
        for (int k = 0; k < kClasses; ++k) {
            c->cls_start[k] = h[8 + k];
            c->cls_total[k] = std::max<int64_t>(1, h[9 + k] - h[8 + k]);
        }
    }
    c->tasks_ready = true;
    return GC_OK;
}

// Launch every class kernel for owner `owner` of `parts`.
template <bool SUP>
static int launch_classes(gc_ctx* c, int owner, int parts, unsigned long long* count, uint32_t* sup,
                          uint16_t* uw16) {
    KArgs a{};
    a.in_pos = c->in_pos.as<int32_t>();
    a.in_src = c->in_src.as<int32_t>();
    a.in_dst = c->in_dst.as<int32_t>();
    a.in_cost = c->in_cost.as<int64_t>();
    a.dag_ptr = c->dag_ptr.as<int64_t>();
    a.dag_col = c->dag_col.as<int32_t>();
    a.total_cost = c->total_cost;
    a.parts = parts;
    a.owner = owner;
    a.sup = sup;
    a.uw16 = uw16;
    a.count = count;
    a.bm_bits = bm_bits_of(c);
    a.long_seg = c->long_seg;
    a.batch = c->block_batch;
    a.uw = c->sup_skip;
    a.huge_max = c->huge_max;
    const uint64_t* tasks = c->task_i0.as<uint64_t>();
    // The warp-task classes (1, 0) run on a side stream forked from the
    // context stream, so they fill the SMs the block-task kernels (3, 2)
    // leave idle at their tails; the context stream joins it before return.
    const bool fork = c->overlap && c->side && (c->ntask[3] > 0 || c->ntask[2] > 0 || c->ntask[4] > 0) &&
                      (c->ntask[1] > 0 || c->ntask[0] > 0);
    cudaStream_t ws = fork ? c->side : c->stream;
    if (fork) {
        GC_CUDA(c, cudaEventRecord(c->ev_fork, c->stream));
        GC_CUDA(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    }
    // Per-context launch cache (the context is bound to one device; the
    // shared-memory opt-in and the occupancy grid are per device and kernel).
    auto prep = [&](int slot, auto kernel, size_t smem, int threads) -> int {
        int& g = c->launch_grid[slot][SUP];
        if (g == 0) {
            if (smem > 48 * 1024 &&
                cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return -1;
            g = occupancy_grid(kernel, smem, threads);
        }
        return g;
    };
    // classes 3 and 2 first (heaviest tasks), then 1, 0
    unsigned long long* next = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 640);   // classes 3, 2
    if (GC_DYN_BATCH) GC_CUDA(c, cudaMemsetAsync(next, 0, 16, c->stream));
    GC_TRY(ensure(c, c->batch_slot, 3 * 2 * 4096 * sizeof(long long)));   // classes 3, 2, 4; grid <= 4096
    long long* slots = c->batch_slot.as<long long>();
    unsigned long long* next4 = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 448);   // class 4
    if (GC_DYN_BATCH) GC_CUDA(c, cudaMemsetAsync(next4, 0, 8, c->stream));
    if (c->ntask[3] > 0) {
        a.next = GC_DYN_BATCH ? next : nullptr;
        a.slot = slots;
        a.tasks = tasks + c->task_off[3];
        a.ntask = c->ntask[3];
        a.task_pref = parts > 1 ? c->task_pref.as<int64_t>() + c->task_off[3] : nullptr;
        a.cls_start = c->cls_start[3];
        a.cls_total = c->cls_total[3];
        const size_t smem = (SUP ? 3 * kTS3 : kTS3) * sizeof(uint32_t);
        constexpr int threads = 32 * GC_HUGE_WARPS(SUP);
        const int grid = prep(3, k_tc_block<SUP, true>, smem, threads);
        if (grid < 0) return cuda_fail(c, cudaGetLastError(), "cudaFuncSetAttribute(k_tc_block huge)", __FILE__, __LINE__);
        GC_LAUNCH(c, (k_tc_block<SUP, true>), (int)std::min<int64_t>({grid, a.ntask, 4096}), threads, smem, a);
    }
    if (c->ntask[4] > 0) {
        // class 4: the bitmap kernel with 8192 (v,w) counters (support); the count
        // pass needs no counters and runs these heads in the class-2 count kernel
        a.next = GC_DYN_BATCH ? next4 : nullptr;
        a.slot = slots + 2 * 2 * 4096;
        a.tasks = tasks + c->task_off[4];
        a.ntask = c->ntask[4];
        a.task_pref = parts > 1 ? c->task_pref.as<int64_t>() + c->task_off[4] : nullptr;
        a.cls_start = c->cls_start[4];
        a.cls_total = c->cls_total[4];
        if (SUP) {
            const size_t smem = (size_t)(kBWS + kBW / 4 + kD4) * sizeof(uint32_t);
            constexpr int threads = 32 * GC_SUP_WARPS;
            const int grid = prep(4, k_tc_block<SUP, false, kD4>, smem, threads);
            if (grid < 0) return cuda_fail(c, cudaGetLastError(), "cudaFuncSetAttribute(k_tc_block wide)", __FILE__, __LINE__);
            GC_LAUNCH(c, (k_tc_block<SUP, false, kD4>), (int)std::min<int64_t>({grid, a.ntask, 4096}), threads, smem, a);
        } else {
            const size_t smem = (size_t)kBWS * sizeof(uint32_t);
            constexpr int threads = 32 * GC_TC_WARPS;
            const int grid = prep(2, k_tc_block<SUP, false>, smem, threads);
            if (grid < 0) return cuda_fail(c, cudaGetLastError(), "cudaFuncSetAttribute(k_tc_block)", __FILE__, __LINE__);
            GC_LAUNCH(c, (k_tc_block<SUP, false>), (int)std::min<int64_t>({grid, a.ntask, 4096}), threads, smem, a);
        }
    }
    if (c->ntask[2] > 0) {
        a.next = GC_DYN_BATCH ? next + 1 : nullptr;
        a.slot = slots + 2 * 4096;
        a.tasks = tasks + c->task_off[2];
        a.ntask = c->ntask[2];
        a.task_pref = parts > 1 ? c->task_pref.as<int64_t>() + c->task_off[2] : nullptr;
        a.cls_start = c->cls_start[2];
        a.cls_total = c->cls_total[2];
        const size_t smem = (SUP ? kBWS + kBW / 4 + kD2 : kBWS) * sizeof(uint32_t);
        constexpr int threads = 32 * (SUP ? GC_SUP_WARPS : GC_TC_WARPS);
        const int grid = prep(2, k_tc_block<SUP, false>, smem, threads);
        if (grid < 0) return cuda_fail(c, cudaGetLastError(), "cudaFuncSetAttribute(k_tc_block)", __FILE__, __LINE__);
        GC_LAUNCH(c, (k_tc_block<SUP, false>), (int)std::min<int64_t>({grid, a.ntask, 4096}), threads, smem, a);
    }
    if (c->ntask[1] > 0) {
        a.tasks = tasks + c->task_off[1];
        a.ntask = c->ntask[1];
        a.task_pref = parts > 1 ? c->task_pref.as<int64_t>() + c->task_off[1] : nullptr;
        a.cls_start = c->cls_start[1];
        a.cls_total = c->cls_total[1];
        const size_t smem = kWarps * (SUP ? 3 * kTS1 : kTS1) * sizeof(uint32_t);
        const int grid = prep(1, k_tc_warp<kTS1, SUP>, smem, 256);
        if (grid < 0) return cuda_fail(c, cudaGetLastError(), "cudaFuncSetAttribute(k_tc_warp)", __FILE__, __LINE__);
        GC_LAUNCH_S(c, ws, (k_tc_warp<kTS1, SUP>), (int)std::min<int64_t>(grid, (a.ntask + kWarps - 1) / kWarps), 256,
                    smem, a);
    }
    if (c->ntask[0] > 0) {
        a.tasks = tasks + c->task_off[0];
        a.ntask = c->ntask[0];
        a.task_pref = parts > 1 ? c->task_pref.as<int64_t>() + c->task_off[0] : nullptr;
        a.cls_start = c->cls_start[0];
        a.cls_total = c->cls_total[0];
        const int grid = prep(0, k_tc_tiny<SUP>, 0, 256);
        GC_LAUNCH_S(c, ws, (k_tc_tiny<SUP>), (int)std::min<int64_t>(grid, (a.ntask + 255) / 256), 256, 0, a);
    }
    if (fork) {
        GC_CUDA(c, cudaEventRecord(c->ev_join, c->side));
        GC_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    }
    return GC_OK;
}

template <bool SUP>
static int run_all_parts(gc_ctx* c, unsigned long long* count, uint32_t* sup, uint16_t* uw16) {
    if (!c->tasks_ready) GC_TRY(prepare_tasks(c));
    const int parts = c->task_parts;
    if (c->total_cost == 0) return GC_OK;
    if (c->loop_parts > 0) {
        // per virtual rank device time (stats.part_ms): the balance of the 1D cut
        const int nt = c->timing ? std::min(parts, 16) : 0;
        for (int r = 0; r <= nt; ++r)
            if (!c->pev[r]) GC_CUDA(c, cudaEventCreate(&c->pev[r]));
        for (int r = 0; r < parts; ++r) {
            if (r < nt) GC_CUDA(c, cudaEventRecord(c->pev[r], c->stream));
            GC_TRY(launch_classes<SUP>(c, r, parts, count, sup, uw16));
        }
        if (nt > 0) {
            GC_CUDA(c, cudaEventRecord(c->pev[nt], c->stream));
            GC_CUDA(c, cudaEventSynchronize(c->pev[nt]));
            for (int r = 0; r < 16; ++r) {
                float ms = 0.f;
                if (r < nt && cudaEventElapsedTime(&ms, c->pev[r], c->pev[r + 1]) != cudaSuccess) {
                    cudaGetLastError();
                    ms = 0.f;
                }
                c->stats.part_ms[r] = r < nt ? ms : 0.0;
            }
        }
    } else {
        GC_TRY(launch_classes<SUP>(c, c->rank, parts, count, sup, uw16));
    }
    return GC_OK;
}

int triangle_count(gc_ctx* c, uint64_t* out) {
    GC_TRY(ensure(c, c->scal, 1024));
    GC_TRY(host_scratch(c, 4096));
    unsigned long long* count = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 192);
    GC_TRY(record(c, 2));
    GC_CUDA(c, cudaMemsetAsync(count, 0, 8, c->stream));
    GC_TRY(record(c, 6));
    GC_TRY(run_all_parts<false>(c, count, nullptr, nullptr));
    GC_TRY(record(c, 7));
    if (c->nccl) GC_TRY(allreduce_u64(c, reinterpret_cast<uint64_t*>(count), 1));
    GC_TRY(record(c, 3));
    GC_TRY(read_small(c, c->hpin, count, 8));
    GC_TRY(sync(c));
    *out = *static_cast<uint64_t*>(c->hpin);
    c->stats.tc_ms = elapsed(c, 2, 3);
    c->stats.tc_kernel_ms = elapsed(c, 6, 7);
    return GC_OK;
}

int support_dag(gc_ctx* c) {
    const int64_t m = c->m;
    GC_TRY(ensure(c, c->sup, (size_t)m * 4));
    GC_TRY(ensure(c, c->scal, 1024));
    unsigned long long* count = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 200);
    GC_CUDA(c, cudaMemsetAsync(c->sup.p, 0, (size_t)m * 4, c->stream));
    GC_CUDA(c, cudaMemsetAsync(count, 0, 8, c->stream));
    uint16_t* uw16 = nullptr;
    if (GC_UW16 && m > 0) {
        // d+(x) <= sqrt(2m) (x's higher-ranked neighbours all have degree >= d+(x)), so with
        // m < 2^31 every (u,w) count is below 2^16 and the 16-bit lanes never carry
        if (c->stats.max_out_degree > 65535) return fail(c, GC_ERR_RANGE, "support pass: d+ above 65535");
        const size_t bytes = (size_t)((m + 3) / 4) * 8;   // whole 64-bit words
        GC_TRY(ensure(c, c->uw16, bytes));
        GC_CUDA(c, cudaMemsetAsync(c->uw16.p, 0, bytes, c->stream));
        uw16 = c->uw16.as<uint16_t>();
    }
    GC_TRY(record(c, 6));
    GC_TRY(run_all_parts<true>(c, count, c->sup.as<uint32_t>(), uw16));
    if (uw16) GC_LAUNCH(c, k_fold_uw, grid_for((m + 3) / 4), kThreads, 0, c->sup.as<uint32_t>(), uw16, m);
    GC_TRY(record(c, 7));
    if (c->nccl) GC_TRY(allreduce_u32(c, c->sup.as<uint32_t>(), (size_t)m));
    return GC_OK;
}

unsigned long long* support_hits(gc_ctx* c) {   // triangles found by the last support pass (device)
    return reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 200);
}

// DAG order -> canonical order.  The canonical ids of consecutive DAG
// positions are scattered over the whole output, so a direct scatter writes a
// partial 32-byte sector per element (C4 supports: 7.3 ms).  Large m first
// sorts the (id, value) pairs on the ids' top 8 bits (one radix pass), then
// scatters with one element per thread and no grid-stride loop: blocks start
// in order, so the writes in flight fall in a few MB of the output and merge
// into full sectors in L2 (a grid-stride loop lets blocks drift apart and
// spreads the writes again: 10 ms against 1.4 ms in scripts/micro).
template <class T>
__global__ void k_scatter_sorted(const uint32_t* __restrict__ idx, const T* __restrict__ vals, int64_t m,
                                 T* __restrict__ out) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < m) out[idx[p]] = vals[p];
}

template <class T>
static int scatter_canonical(gc_ctx* c, const T* dag_vals, T* out) {
    const int64_t m = c->m;
    if (m == 0) return GC_OK;
    const int B = ceil_log2_u64((uint64_t)m);
    if (m < ((int64_t)1 << 22) || B > 31) {
        GC_LAUNCH(c, k_scatter_t<T>, grid_for(m), kThreads, 0, dag_vals, c->dag_eid.as<int32_t>(), m, out);
        return GC_OK;
    }
    GC_TRY(ensure(c, c->keys_a, (size_t)m * 4));   // build / task-preparation scratch, free here
    GC_TRY(ensure(c, c->keys_b, (size_t)m * sizeof(T)));
    uint32_t* ks = reinterpret_cast<uint32_t*>(c->keys_a.p);
    T* vs = reinterpret_cast<T*>(c->keys_b.p);
    const uint32_t* eid = reinterpret_cast<const uint32_t*>(c->dag_eid.p);
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, eid, ks, dag_vals, vs, m, B - 8, B, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, eid, ks, dag_vals, vs, m, B - 8, B, c->stream));
    c->stats.lib_launches += 3;
    GC_LAUNCH(c, k_scatter_sorted<T>, (int)((m + kThreads - 1) / kThreads), kThreads, 0, ks, vs, m, out);
    return GC_OK;
}

int scatter_canonical_u32(gc_ctx* c, const uint32_t* dag_vals, uint32_t* out) {
    return scatter_canonical<uint32_t>(c, dag_vals, out);
}
int scatter_canonical_u8(gc_ctx* c, const uint8_t* dag_vals, uint8_t* out) {
    return scatter_canonical<uint8_t>(c, dag_vals, out);
}

}  // namespace gcx
