// build_csr.cu — on-GPU graph construction.
//
//  a2  canonicalise: drop self loops, fold both orientations to (min, max),
//      radix-sort the packed keys on 2b bits (b = id bits), unique
//      (P:134-136 [Data Sets]: "all self loops were removed", "additional
//      edges in the opposite direction were added"; reading A1: dedup).
//  a3  degrees d(x) (Alg. 4 "d = sum(E)").
//  a4  rank r(x) = position of (d(x), x) in lexicographic order; relabel
//      every vertex by its rank and orient each edge low -> high rank.  In
//      rank space the oriented graph is the strict upper triangle U of the
//      relabelled A (Alg. 3's (L, U) <- A), whose rows are sorted and
//      short: d+(x) <= sqrt(2m).  Also the transposed lists (in-lists) that
//      the intersection kernels walk, grouped by head vertex.
//
// Radix sorts are CUB's (library primitive); everything else is ours.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>

#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "gc_internal.cuh"

#ifndef GC_SPLIT_SORT1
#define GC_SPLIT_SORT1 1   // canonicalisation sort as two 32-bit pair sorts (hi, then lo)
#endif

namespace gcx {

namespace {

__global__ void k_scan_ids(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t nnz,
                           int* __restrict__ maxid, int* __restrict__ neg) {
    int mx = -1, ng = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        int a = __ldg(u + i), b = __ldg(v + i);
        mx = max(mx, max(a, b));
        ng |= (a < 0) | (b < 0);
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    ng = __reduce_or_sync(0xffffffffu, (unsigned)ng);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(maxid, mx);
        if (ng) atomicOr(neg, 1);
    }
}

// key = (min << b) | max ; self loops -> sentinel (all ones in the low 2b bits,
// never a real key since it would need min == max).
__global__ void k_pack(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t nnz, int b,
                       uint64_t sent, uint64_t* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t a = (uint32_t)__ldg(u + i), c = (uint32_t)__ldg(v + i);
        uint32_t lo = min(a, c), hi = max(a, c);
        keys[i] = (a == c) ? sent : (((uint64_t)lo << b) | hi);
    }
}

// Degrees from the canonical list (sorted by (lo, hi)): the lo side is the
// length of each lo run (its bounds written, no atomics), the hi side one
// atomic per edge.
// split keys for the canonicalisation sort: lo = min, hi = max as two 32-bit
// arrays; a self loop becomes (2^b - 1, 2^b - 1), which sorts last and is no
// real edge (lo < hi for every real one)
__global__ void k_pack_split(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t nnz, uint32_t sent,
                             uint32_t* __restrict__ lo_out, uint32_t* __restrict__ hi_out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = (uint32_t)__ldg(u + i), c = (uint32_t)__ldg(v + i);
        lo_out[i] = a == c ? sent : min(a, c);
        hi_out[i] = a == c ? sent : max(a, c);
    }
}

// (lo, hi) halves of the sorted pairs -> the canonical 64-bit key, on the fly
struct JoinKey {
    const uint32_t* lo;
    const uint32_t* hi;
    int b;
    __host__ __device__ uint64_t operator()(int64_t i) const { return ((uint64_t)lo[i] << b) | hi[i]; }
};


__global__ void k_degrees(const uint64_t* __restrict__ canon, int64_t m, int b, int32_t* __restrict__ deg,
                          int32_t* __restrict__ first, int32_t* __restrict__ last) {
    const uint64_t mask = (1ULL << b) - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = canon[e];
        const uint32_t lo = (uint32_t)(k >> b);
        atomicAdd(deg + (k & mask), 1);
        if (e == 0 || (uint32_t)(canon[e - 1] >> b) != lo) first[lo] = (int32_t)e;
        if (e == m - 1 || (uint32_t)(canon[e + 1] >> b) != lo) last[lo] = (int32_t)(e + 1);
    }
}

__global__ void k_degrees_lo(const int32_t* __restrict__ first, const int32_t* __restrict__ last, int64_t n,
                             int32_t* __restrict__ deg) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
        deg[x] += last[x] - first[x];
}

// vertex sort keys: the degree alone, ids as payload (a stable radix sort of
// ascending ids by degree is the (degree, id) order)
__global__ void k_vkeys(const int32_t* __restrict__ deg, int64_t n, uint32_t* __restrict__ keys,
                        int32_t* __restrict__ ids, int* __restrict__ maxdeg) {
    int mx = 0;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int d = deg[x];
        keys[x] = (uint32_t)d;
        ids[x] = (int32_t)x;
        mx = max(mx, d);
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) atomicMax(maxdeg, mx);
}

__global__ void k_rank_scatter(const int32_t* __restrict__ sorted_ids, int64_t n, int32_t* __restrict__ rank_of) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        rank_of[sorted_ids[r]] = (int32_t)r;
}

// oriented key in rank space: (lo << b) | hi with lo = min rank, hi = max rank
__global__ void k_orient(const uint64_t* __restrict__ canon, int64_t m, int b, const int32_t* __restrict__ rank_of,
                         uint64_t* __restrict__ dkeys, int32_t* __restrict__ iota) {
    const uint64_t mask = (1ULL << b) - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = canon[e];
        uint32_t ra = (uint32_t)__ldg(rank_of + (k >> b)), rb = (uint32_t)__ldg(rank_of + (k & mask));
        uint32_t lo = min(ra, rb), hi = max(ra, rb);
        dkeys[e] = ((uint64_t)lo << b) | hi;
        iota[e] = (int32_t)e;
    }
}

// split of the sorted oriented keys fused with the row bounds of the CSR
// (first / last position of each row, rows = high part)
__global__ void k_split_keys_bounds(const uint64_t* __restrict__ keys, int64_t m, int b, int32_t* __restrict__ col,
                                    int32_t* __restrict__ row, int32_t* __restrict__ first,
                                    int32_t* __restrict__ last) {
    const uint64_t mask = (1ULL << b) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        const int32_t r = (int32_t)(k >> b);
        row[i] = r;
        col[i] = (int32_t)(k & mask);
        if (i == 0 || (int32_t)(keys[i - 1] >> b) != r) first[r] = (int32_t)i;
        if (i == m - 1 || (int32_t)(keys[i + 1] >> b) != r) last[r] = (int32_t)(i + 1);
    }
}


// CSR row pointers from a row-sorted COO row array, in three parallel steps
// (no thread walks a gap of empty rows): each run of equal rows records its
// bounds, the row lengths are formed, and an exclusive scan gives ptr.
__global__ void k_run_bounds(const int32_t* __restrict__ row, int64_t m, int32_t* __restrict__ first,
                             int32_t* __restrict__ last) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = row[i];
        if (i == 0 || row[i - 1] != r) first[r] = (int32_t)i;
        if (i == m - 1 || row[i + 1] != r) last[r] = (int32_t)(i + 1);
    }
}

__global__ void k_row_len(const int32_t* __restrict__ first, const int32_t* __restrict__ last, int64_t n,
                          int64_t* __restrict__ len) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n; x += (int64_t)gridDim.x * blockDim.x)
        len[x] = (x < n) ? (int64_t)(last[x] - first[x]) : 0;
}


// in-list sort payload: (tail << 32) | DAG position, so the sort carries the
// tail along (no gather afterwards)
__global__ void k_pos_tail(const int32_t* __restrict__ dag_src, int64_t m, uint64_t* __restrict__ vals) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x)
        vals[p] = ((uint64_t)(uint32_t)dag_src[p] << 32) | (uint64_t)(uint32_t)p;
}

__global__ void k_split_pos_tail_bounds(const uint64_t* __restrict__ vals, const int32_t* __restrict__ head, int64_t m,
                                        int32_t* __restrict__ pos, int32_t* __restrict__ tail,
                                        int32_t* __restrict__ first, int32_t* __restrict__ last) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x = vals[i];
        pos[i] = (int32_t)(uint32_t)x;
        tail[i] = (int32_t)(x >> 32);
        const int32_t r = head[i];
        if (i == 0 || head[i - 1] != r) first[r] = (int32_t)i;
        if (i == m - 1 || head[i + 1] != r) last[r] = (int32_t)(i + 1);
    }
}


// Work-model sums over vertices: wedges = Σ C(d+,2), Q_out = Σ d+², Q_in = Σ d- d+,
// max d+, max d.
// Also (aux) heads with d+ > 256: rank span of N+(x) in buckets <= 2^17, 2^18,
// 2^19, more — counts in acc[5..8], in-degree-weighted in acc[9..12].
__global__ void k_graph_stats(const int64_t* __restrict__ dag_ptr, const int64_t* __restrict__ in_ptr,
                              const int32_t* __restrict__ deg, const int32_t* __restrict__ dag_col, int64_t n,
                              unsigned long long* __restrict__ acc) {
    unsigned long long w = 0, qo = 0, qi = 0;
    int mo = 0, md = 0;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long dp = (unsigned long long)(dag_ptr[x + 1] - dag_ptr[x]);
        unsigned long long dm = (unsigned long long)(in_ptr[x + 1] - in_ptr[x]);
        w += dp * (dp - (dp > 0)) / 2;
        qo += dp * dp;
        qi += dm * dp;
        mo = max(mo, (int)dp);
        md = max(md, deg[x]);
        if (dp > 256) {
            const int64_t span = (int64_t)dag_col[dag_ptr[x + 1] - 1] - x;
            const int bkt = span <= (1 << 17) ? 0 : span <= (1 << 18) ? 1 : span <= (1 << 19) ? 2 : 3;
            atomicAdd(acc + 5 + bkt, 1ULL);
            atomicAdd(acc + 9 + bkt, dm);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        w += __shfl_xor_sync(0xffffffffu, w, o);
        qo += __shfl_xor_sync(0xffffffffu, qo, o);
        qi += __shfl_xor_sync(0xffffffffu, qi, o);
    }
    mo = __reduce_max_sync(0xffffffffu, mo);
    md = __reduce_max_sync(0xffffffffu, md);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc + 0, w);
        atomicAdd(acc + 1, qo);
        atomicAdd(acc + 2, qi);
        atomicMax(acc + 3, (unsigned long long)mo);
        atomicMax(acc + 4, (unsigned long long)md);
    }
}

__global__ void k_unpack_canon(const uint64_t* __restrict__ canon, int64_t m, int b, int32_t* __restrict__ u,
                               int32_t* __restrict__ v) {
    const uint64_t mask = (1ULL << b) - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = canon[e];
        u[e] = (int32_t)(k >> b);
        v[e] = (int32_t)(k & mask);
    }
}

// ---- partitioned build: per-owner selection kernels
// raw pairs of owner range lo in [Llo, Lhi) as split (lo, hi) halves; order
// of appends arbitrary (the pair sorts order them fully)
__global__ void k_pack_range(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t nnz, uint32_t Llo,
                             uint32_t Lhi, uint32_t* __restrict__ lo_out, uint32_t* __restrict__ hi_out,
                             unsigned long long* __restrict__ count) {
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < nnz; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        uint32_t lo = 0, hi = 0;
        bool in = false;
        if (i < nnz) {
            const uint32_t a = (uint32_t)__ldg(u + i), c = (uint32_t)__ldg(v + i);
            lo = min(a, c);
            hi = max(a, c);
            in = a != c && lo >= Llo && lo < Lhi;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        unsigned long long base = 0;
        if (lane == 0 && bal) base = atomicAdd(count, (unsigned long long)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (in) {
            const unsigned long long o = base + __popc(bal & ((1u << lane) - 1));
            lo_out[o] = lo;
            hi_out[o] = hi;
        }
    }
}

// out-degree of every tail (lower rank) of the canonical edges
__global__ void k_tail_count(const uint64_t* __restrict__ canon, int64_t m, int b, const int32_t* __restrict__ rank_of,
                             unsigned long long* __restrict__ cnt) {
    const uint64_t mask = (1ULL << b) - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = canon[e];
        const uint32_t ra = (uint32_t)__ldg(rank_of + (k >> b)), rb = (uint32_t)__ldg(rank_of + (k & mask));
        atomicAdd(cnt + min(ra, rb), 1ULL);
    }
}

// in-degree of every head (lanes with the same head add once)
__global__ void k_head_count(const int32_t* __restrict__ dag_col, int64_t m, unsigned long long* __restrict__ cnt) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t h = dag_col[p];
        const unsigned grp = __match_any_sync(__activemask(), h);
        if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(cnt + h, (unsigned long long)__popc(grp));
    }
}

// owner cut points: cut[r] = first row x with ptr[x] >= r * total / parts (r = 0..parts)
__global__ void k_cuts(const int64_t* __restrict__ ptr, int64_t n, int parts, int64_t* __restrict__ cut) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > parts) return;
    const int64_t total = ptr[n];
    const int64_t want = (int64_t)((__int128)total * r / parts);
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ptr[mid] < want) lo = mid + 1; else hi = mid;
    }
    cut[r] = r == parts ? n : lo;
}

// canonical edges whose tail lies in [Tlo, Thi): oriented key + canonical id
struct TailInRange {
    const uint64_t* canon;
    const int32_t* rank_of;
    int b;
    uint32_t Tlo, Thi;
    __device__ bool operator()(int32_t e) const {
        const uint64_t k = canon[e];
        const uint32_t ra = (uint32_t)rank_of[k >> b], rb = (uint32_t)rank_of[k & ((1ULL << b) - 1)];
        const uint32_t t = min(ra, rb);
        return t >= Tlo && t < Thi;
    }
};

__global__ void k_orient_sel(const uint64_t* __restrict__ canon, const int32_t* __restrict__ sel, int64_t cnt, int b,
                             const int32_t* __restrict__ rank_of, uint64_t* __restrict__ keys) {
    const uint64_t mask = (1ULL << b) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = canon[sel[i]];
        const uint32_t ra = (uint32_t)__ldg(rank_of + (k >> b)), rb = (uint32_t)__ldg(rank_of + (k & mask));
        keys[i] = ((uint64_t)min(ra, rb) << b) | max(ra, rb);
    }
}

__global__ void k_split_keys(const uint64_t* __restrict__ keys, int64_t cnt, int b, int32_t* __restrict__ col,
                             int32_t* __restrict__ row) {
    const uint64_t mask = (1ULL << b) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        row[i] = (int32_t)(k >> b);
        col[i] = (int32_t)(k & mask);
    }
}

struct HeadInRange {
    const int32_t* dag_col;
    int32_t Hlo, Hhi;
    __device__ bool operator()(int32_t p) const {
        const int32_t h = dag_col[p];
        return h >= Hlo && h < Hhi;
    }
};

__global__ void k_gather_heads(const int32_t* __restrict__ sel, int64_t cnt, const int32_t* __restrict__ dag_col,
                               uint32_t* __restrict__ heads) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        heads[i] = (uint32_t)dag_col[sel[i]];
}

__global__ void k_in_tail(const int32_t* __restrict__ pos, int64_t cnt, const int32_t* __restrict__ dag_src,
                          int32_t* __restrict__ tail) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        tail[i] = dag_src[pos[i]];
}

}  // namespace

// Sort keys (and optional int32 payload) on bits [0, nbits); results in
// keys_out / vals_out.
// ptr[x] = first i with row[i] >= x, for a row-sorted array of length m.
// Scratch: keys_a (first/last, 8n bytes), keys_b (lengths, 8(n+1) bytes).
static int csr_ptr_from_sorted(gc_ctx* c, const int32_t* row, int64_t m, int64_t n, int64_t* ptr) {
    GC_TRY(ensure(c, c->keys_a, (size_t)(n + 1) * 8));
    GC_TRY(ensure(c, c->keys_b, (size_t)(n + 1) * 8));
    int32_t* first = reinterpret_cast<int32_t*>(c->keys_a.p);
    int32_t* last = first + n;
    int64_t* len = c->keys_b.as<int64_t>();
    GC_CUDA(c, cudaMemsetAsync(first, 0, (size_t)n * 8, c->stream));
    if (m > 0) GC_LAUNCH(c, k_run_bounds, grid_for(m), kThreads, 0, row, m, first, last);
    GC_LAUNCH(c, k_row_len, grid_for(n + 1), kThreads, 0, first, last, n, len);
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, len, ptr, n + 1, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, len, ptr, n + 1, c->stream));
    c->stats.lib_launches += 2;
    return GC_OK;
}

// row pointers from first / last bounds already written (rows without entries: first = last = 0)
static int ptr_from_bounds(gc_ctx* c, const int32_t* first, const int32_t* last, int64_t n, int64_t* len,
                           int64_t* ptr) {
    GC_LAUNCH(c, k_row_len, grid_for(n + 1), kThreads, 0, first, last, n, len);
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, len, ptr, n + 1, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, len, ptr, n + 1, c->stream));
    c->stats.lib_launches += 2;
    return GC_OK;
}

static int radix_sort(gc_ctx* c, const uint64_t* kin, uint64_t* kout, const int32_t* vin, int32_t* vout, int64_t N,
                      int nbits) {
    if (N <= 0) return GC_OK;
    size_t tmp = 0;
    if (vin) {
        GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, N, 0, nbits, c->stream));
    } else {
        GC_CUDA(c, cub::DeviceRadixSort::SortKeys(nullptr, tmp, kin, kout, N, 0, nbits, c->stream));
    }
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    if (vin) {
        GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, kin, kout, vin, vout, N, 0, nbits, c->stream));
    } else {
        GC_CUDA(c, cub::DeviceRadixSort::SortKeys(c->cub_tmp.p, tmp, kin, kout, N, 0, nbits, c->stream));
    }
    c->stats.lib_launches += 2 + (nbits + 7) / 8;   // histogram + scan + one onesweep pass per digit
    return GC_OK;
}

// ------------------------------------------------------ partitioned build --
// the three sorts of the build are cut between the owners
// (NCCL ranks, or loopback virtual ranks on one GPU): owner r sorts only the
// raw pairs whose low endpoint falls in its id range, the oriented edges whose
// tail falls in its rank range, and the in-edges whose head falls in its
// rank range (ranges cut at equal edge counts from the replicated row
// pointers); the sorted parts are concatenated on every rank (NCCL: a
// variable-size allgather per array).  The O(n) / O(m) counting passes
// (degrees, row pointers, cut points) stay replicated.
static int build_owners(const gc_ctx* c) {
    if (c->loop_parts > 1) return c->loop_parts;
    return c->nccl ? c->nranks : 1;
}
static bool part_build(const gc_ctx* c) {
    if (c->build_part >= 0) return c->build_part == 1;
    return build_owners(c) > 1;
}

// per-owner device time of the partitioned stages (loopback: stats.part_build_ms)
struct OwnerTimer {
    gc_ctx* c;
    bool on;
    int nt;
    explicit OwnerTimer(gc_ctx* cc) : c(cc), on(cc->timing && cc->loop_parts > 1), nt(std::min(cc->loop_parts, 16)) {}
    int begin(int r) {
        if (!on || r >= nt) return GC_OK;
        if (!c->pev[r]) GC_CUDA(c, cudaEventCreate(&c->pev[r]));
        if (!c->pev[16]) GC_CUDA(c, cudaEventCreate(&c->pev[16]));
        GC_CUDA(c, cudaEventRecord(c->pev[r], c->stream));
        return GC_OK;
    }
    int end(int r) {
        if (!on || r >= nt) return GC_OK;
        GC_CUDA(c, cudaEventRecord(c->pev[16], c->stream));
        GC_CUDA(c, cudaEventSynchronize(c->pev[16]));
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->pev[r], c->pev[16]) != cudaSuccess) cudaGetLastError();
        c->stats.part_build_ms[r] += ms;
        return GC_OK;
    }
};

template <class Pred>
static int select_iota(gc_ctx* c, int64_t N, Pred pred, int32_t* out, int64_t* d_count) {
    thrust::counting_iterator<int32_t> iota(0);
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceSelect::If(nullptr, tmp, iota, out, d_count, N, pred, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceSelect::If(c->cub_tmp.p, tmp, iota, out, d_count, N, pred, c->stream));
    c->stats.lib_launches += 2;
    return GC_OK;
}

// cut points of `parts` owners over row pointers ptr[0..n] (host copy in cut_h)
static int owner_cuts(gc_ctx* c, const int64_t* ptr, int64_t n, int parts, int64_t* cut_h, int64_t* base_h) {
    GC_TRY(ensure(c, c->tmp_b, (size_t)(parts + 1) * 8));
    int64_t* cut = c->tmp_b.as<int64_t>();
    GC_LAUNCH(c, k_cuts, 1, 128, 0, ptr, n, parts, cut);
    int64_t* h = static_cast<int64_t*>(c->hpin);
    GC_TRY(read_small(c, h, cut, (size_t)(parts + 1) * 8));
    GC_TRY(sync(c));
    for (int r = 0; r <= parts; ++r) cut_h[r] = h[r];
    for (int r = 0; r <= parts; ++r) GC_TRY(read_small(c, h + 128 + r, ptr + cut_h[r], 8));
    GC_TRY(sync(c));
    for (int r = 0; r <= parts; ++r) base_h[r] = h[128 + r];
    return GC_OK;
}

// a2 across owners: canon = concatenation of the owners' sorted unique parts
static int part_canonical(gc_ctx* c, int64_t nnz, int64_t n, int b, int64_t* m_out) {
    const int P = build_owners(c);
    const bool nccl = c->nccl != nullptr;
    const int r0 = nccl ? c->rank : 0, r1 = nccl ? c->rank + 1 : P;
    int64_t* h = static_cast<int64_t*>(c->hpin);
    uint32_t* lo_a = reinterpret_cast<uint32_t*>(c->keys_a.p);
    uint32_t* hi_a = lo_a + nnz;
    uint32_t* lo_b = reinterpret_cast<uint32_t*>(c->keys_b.p);
    uint32_t* hi_b = lo_b + nnz;
    GC_TRY(ensure(c, c->canon, (size_t)nnz * 8));
    GC_TRY(ensure(c, c->tmp_a, (size_t)nnz * 8 + 8));
    uint64_t* part = c->tmp_a.as<uint64_t>();               // this owner's unique keys
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 960);
    int64_t* d_nsel = reinterpret_cast<int64_t*>(c->scal.as<char>() + 968);
    OwnerTimer tm(c);
    int64_t off = 0, mine = 0;
    for (int r = r0; r < r1; ++r) {
        GC_TRY(tm.begin(r));
        const uint32_t Llo = (uint32_t)(n * r / P), Lhi = (uint32_t)(n * (r + 1) / P);
        GC_CUDA(c, cudaMemsetAsync(cnt, 0, 8, c->stream));
        GC_LAUNCH(c, k_pack_range, grid_for(nnz), kThreads, 0, c->raw_u.as<int32_t>(), c->raw_v.as<int32_t>(), nnz,
                  Llo, Lhi, lo_a, hi_a, cnt);
        GC_TRY(read_small(c, h, cnt, 8));
        GC_TRY(sync(c));
        const int64_t k = h[0];
        int64_t mr = 0;
        if (k > 0) {
            size_t tmp = 0;
            GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, hi_a, hi_b, lo_a, lo_b, k, 0, b, c->stream));
            GC_TRY(ensure(c, c->cub_tmp, tmp));
            tmp = c->cub_tmp.cap;
            GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, hi_a, hi_b, lo_a, lo_b, k, 0, b, c->stream));
            GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, lo_b, lo_a, hi_b, hi_a, k, 0, b, c->stream));
            c->stats.lib_launches += 2 * (2 + (b + 7) / 8);
            auto joined = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), JoinKey{lo_a, hi_a, b});
            size_t tmp2 = 0;
            GC_CUDA(c, cub::DeviceSelect::Unique(nullptr, tmp2, joined, part, d_nsel, k, c->stream));
            GC_TRY(ensure(c, c->cub_tmp, tmp2));
            tmp2 = c->cub_tmp.cap;
            GC_CUDA(c, cub::DeviceSelect::Unique(c->cub_tmp.p, tmp2, joined, part, d_nsel, k, c->stream));
            c->stats.lib_launches += 2;
            GC_TRY(read_small(c, h, d_nsel, 8));
            GC_TRY(sync(c));
            mr = h[0];
        }
        if (!nccl && mr > 0)
            GC_CUDA(c, cudaMemcpyAsync(c->canon.as<uint64_t>() + off, part, (size_t)mr * 8, cudaMemcpyDeviceToDevice,
                                       c->stream));
        off += mr;
        mine = mr;
        GC_TRY(tm.end(r));
    }
    if (nccl) {
        // sizes of every rank's part, then the parts (64-bit keys as int32 pairs)
        uint32_t* share = reinterpret_cast<uint32_t*>(c->scal.as<char>() + 704);
        *static_cast<uint32_t*>(c->hpin) = (uint32_t)mine;
        GC_CUDA(c, cudaMemcpyAsync(share + c->rank, c->hpin, 4, cudaMemcpyHostToDevice, c->stream));
        GC_TRY(allgather_u32(c, share + c->rank, share, 1));
        GC_TRY(read_small(c, h, share, (size_t)P * 4));
        GC_TRY(sync(c));
        int64_t counts[64], offs[64];
        off = 0;
        for (int r = 0; r < P; ++r) {
            counts[r] = 2 * (int64_t)reinterpret_cast<uint32_t*>(h)[r];
            offs[r] = off;
            off += counts[r];
        }
        if (mine > 0)
            GC_CUDA(c, cudaMemcpyAsync(c->canon.as<int32_t>() + offs[c->rank], part, (size_t)mine * 8,
                                       cudaMemcpyDeviceToDevice, c->stream));
        GC_TRY(allgatherv_i32(c, c->canon.as<int32_t>(), c->canon.as<int32_t>(), counts, offs));
        off /= 2;
    }
    *m_out = off;
    return GC_OK;
}

// a4 across owners: DAG rows of the tails in each owner's rank range
static int part_orient(gc_ctx* c, int64_t n, int b, int64_t m) {
    const int P = build_owners(c);
    const bool nccl = c->nccl != nullptr;
    const int r0 = nccl ? c->rank : 0, r1 = nccl ? c->rank + 1 : P;
    GC_TRY(ensure(c, c->tmp_a, (size_t)(n + 1) * 8));
    unsigned long long* cnt = c->tmp_a.as<unsigned long long>();
    int64_t* dptr = c->dag_ptr.as<int64_t>();
    GC_CUDA(c, cudaMemsetAsync(cnt, 0, (size_t)(n + 1) * 8, c->stream));
    if (m > 0) GC_LAUNCH(c, k_tail_count, grid_for(m), kThreads, 0, c->canon.as<uint64_t>(), m, b,
                         c->rank_of.as<int32_t>(), cnt);
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, dptr, n + 1, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, cnt, dptr, n + 1, c->stream));
    c->stats.lib_launches += 2;
    int64_t cut[65], base[65];
    GC_TRY(owner_cuts(c, dptr, n, P, cut, base));
    int64_t* d_nsel = reinterpret_cast<int64_t*>(c->scal.as<char>() + 968);
    int32_t* sel = c->vals_a.as<int32_t>();
    uint64_t* ka = c->keys_a.as<uint64_t>();
    uint64_t* kb = c->keys_b.as<uint64_t>();
    OwnerTimer tm(c);
    for (int r = r0; r < r1; ++r) {
        const int64_t k = base[r + 1] - base[r];
        if (k <= 0) continue;
        GC_TRY(tm.begin(r));
        GC_TRY(select_iota(c, m, TailInRange{c->canon.as<uint64_t>(), c->rank_of.as<int32_t>(), b, (uint32_t)cut[r],
                                              (uint32_t)cut[r + 1]},
                           sel, d_nsel));
        GC_LAUNCH(c, k_orient_sel, grid_for(k), kThreads, 0, c->canon.as<uint64_t>(), sel, k, b,
                  c->rank_of.as<int32_t>(), ka);
        GC_TRY(radix_sort(c, ka, kb, sel, c->dag_eid.as<int32_t>() + base[r], k, 2 * b));
        GC_LAUNCH(c, k_split_keys, grid_for(k), kThreads, 0, kb, k, b, c->dag_col.as<int32_t>() + base[r],
                  c->dag_src.as<int32_t>() + base[r]);
        GC_TRY(tm.end(r));
    }
    if (nccl) {
        int64_t counts[64], offs[64];
        for (int r = 0; r < P; ++r) {
            counts[r] = base[r + 1] - base[r];
            offs[r] = base[r];
        }
        GC_TRY(allgatherv_i32(c, c->dag_col.as<int32_t>(), c->dag_col.as<int32_t>(), counts, offs));
        GC_TRY(allgatherv_i32(c, c->dag_src.as<int32_t>(), c->dag_src.as<int32_t>(), counts, offs));
        GC_TRY(allgatherv_i32(c, c->dag_eid.as<int32_t>(), c->dag_eid.as<int32_t>(), counts, offs));
    }
    return GC_OK;
}

// in-lists across owners: the in-edges of the heads in each owner's rank range
static int part_inlists(gc_ctx* c, int64_t n, int b, int64_t m) {
    const int P = build_owners(c);
    const bool nccl = c->nccl != nullptr;
    const int r0 = nccl ? c->rank : 0, r1 = nccl ? c->rank + 1 : P;
    GC_TRY(ensure(c, c->tmp_a, (size_t)(n + 1) * 8));
    unsigned long long* cnt = c->tmp_a.as<unsigned long long>();
    int64_t* iptr = c->in_ptr.as<int64_t>();
    GC_CUDA(c, cudaMemsetAsync(cnt, 0, (size_t)(n + 1) * 8, c->stream));
    if (m > 0) GC_LAUNCH(c, k_head_count, grid_for(m), kThreads, 0, c->dag_col.as<int32_t>(), m, cnt);
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, iptr, n + 1, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, cnt, iptr, n + 1, c->stream));
    c->stats.lib_launches += 2;
    int64_t cut[65], base[65];
    GC_TRY(owner_cuts(c, iptr, n, P, cut, base));
    int64_t* d_nsel = reinterpret_cast<int64_t*>(c->scal.as<char>() + 968);
    int32_t* sel = c->vals_a.as<int32_t>();
    uint32_t* heads = reinterpret_cast<uint32_t*>(c->keys_a.p);
    OwnerTimer tm(c);
    for (int r = r0; r < r1; ++r) {
        const int64_t k = base[r + 1] - base[r];
        if (k <= 0) continue;
        GC_TRY(tm.begin(r));
        // positions ascending (stable selection), then a stable sort on the head: (head, tail) order
        GC_TRY(select_iota(c, m, HeadInRange{c->dag_col.as<int32_t>(), (int32_t)cut[r], (int32_t)cut[r + 1]}, sel,
                           d_nsel));
        GC_LAUNCH(c, k_gather_heads, grid_for(k), kThreads, 0, sel, k, c->dag_col.as<int32_t>(), heads);
        size_t t2 = 0;
        uint32_t* hout = reinterpret_cast<uint32_t*>(c->in_dst.as<int32_t>() + base[r]);
        int32_t* pout = c->in_pos.as<int32_t>() + base[r];
        GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, t2, heads, hout, sel, pout, k, 0, b, c->stream));
        GC_TRY(ensure(c, c->cub_tmp, t2));
        t2 = c->cub_tmp.cap;
        GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, t2, heads, hout, sel, pout, k, 0, b, c->stream));
        c->stats.lib_launches += 2 + (b + 7) / 8;
        GC_LAUNCH(c, k_in_tail, grid_for(k), kThreads, 0, pout, k, c->dag_src.as<int32_t>(),
                  c->in_src.as<int32_t>() + base[r]);
        GC_TRY(tm.end(r));
    }
    if (nccl) {
        int64_t counts[64], offs[64];
        for (int r = 0; r < P; ++r) {
            counts[r] = base[r + 1] - base[r];
            offs[r] = base[r];
        }
        GC_TRY(allgatherv_i32(c, c->in_pos.as<int32_t>(), c->in_pos.as<int32_t>(), counts, offs));
        GC_TRY(allgatherv_i32(c, c->in_src.as<int32_t>(), c->in_src.as<int32_t>(), counts, offs));
        GC_TRY(allgatherv_i32(c, c->in_dst.as<int32_t>(), c->in_dst.as<int32_t>(), counts, offs));
    }
    return GC_OK;
}

int build_csr(gc_ctx* c) {
    const int64_t nnz = c->nnz;
    c->n = 0;
    c->m = 0;
    c->bits = 1;
    GC_TRY(ensure(c, c->scal, 1024));
    int* d_scal = c->scal.as<int>();
    GC_TRY(host_scratch(c, 4096));
    int64_t* h = static_cast<int64_t*>(c->hpin);

    // ---- n = max id + 1; reject negative ids
    GC_CUDA(c, cudaMemsetAsync(d_scal, 0xff, sizeof(int), c->stream));       // maxid = -1
    GC_CUDA(c, cudaMemsetAsync(d_scal + 1, 0, sizeof(int), c->stream));      // neg = 0
    if (nnz > 0)
        GC_LAUNCH(c, k_scan_ids, grid_for(nnz), kThreads, 0, c->raw_u.as<int32_t>(), c->raw_v.as<int32_t>(), nnz,
                  d_scal, d_scal + 1);
    GC_TRY(read_small(c, h, d_scal, 2 * sizeof(int)));
    GC_TRY(sync(c));
    int maxid = reinterpret_cast<int*>(h)[0];
    int neg = reinterpret_cast<int*>(h)[1];
    if (neg) return fail(c, GC_ERR_INVALID, "gc_build_csr: negative vertex id");
    if (maxid == INT32_MAX) return fail(c, GC_ERR_RANGE, "gc_build_csr: vertex id 2^31-1 leaves no room for n");
    const int64_t n = (int64_t)maxid + 1;
    c->n = n;
    const int b = n > 1 ? ceil_log2_u64((uint64_t)n) : 1;
    c->bits = b;

    // ---- a2: pack, sort, unique
    int64_t m = 0;
    const bool part = part_build(c) && b <= 31;
    for (int r = 0; r < 16; ++r) c->stats.part_build_ms[r] = 0.0;
    if (nnz > 0 && part) {
        GC_TRY(ensure(c, c->keys_a, (size_t)nnz * 8));
        GC_TRY(ensure(c, c->keys_b, (size_t)nnz * 8));
        GC_TRY(part_canonical(c, nnz, n, b, &m));
    } else if (nnz > 0) {
        GC_TRY(ensure(c, c->keys_a, (size_t)nnz * 8));
        GC_TRY(ensure(c, c->keys_b, (size_t)nnz * 8));
        const uint64_t sent = (2 * b >= 64) ? ~0ULL : ((1ULL << (2 * b)) - 1);
        bool joined_done = false;
        if (GC_SPLIT_SORT1 && b <= 31) {
            // (lo, hi) order by two stable 32-bit pair sorts, hi then lo: the same
            // bytes per pass as one 64-bit key sort, with 32-bit digits passes
            uint32_t* lo_a = reinterpret_cast<uint32_t*>(c->keys_a.p);
            uint32_t* hi_a = lo_a + nnz;
            uint32_t* lo_b = reinterpret_cast<uint32_t*>(c->keys_b.p);
            uint32_t* hi_b = lo_b + nnz;
            GC_LAUNCH(c, k_pack_split, grid_for(nnz), kThreads, 0, c->raw_u.as<int32_t>(), c->raw_v.as<int32_t>(), nnz,
                      (uint32_t)((1ULL << b) - 1), lo_a, hi_a);
            size_t tmp = 0;
            GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, hi_a, hi_b, lo_a, lo_b, nnz, 0, b, c->stream));
            GC_TRY(ensure(c, c->cub_tmp, tmp));
            tmp = c->cub_tmp.cap;
            GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, hi_a, hi_b, lo_a, lo_b, nnz, 0, b, c->stream));
            GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, lo_b, lo_a, hi_b, hi_a, nnz, 0, b, c->stream));
            c->stats.lib_launches += 2 * (2 + (b + 7) / 8);
            // the unique pass reads the two halves joined on the fly (no 64-bit key array)
            GC_TRY(ensure(c, c->canon, (size_t)nnz * 8));
            int64_t* d_nsel = reinterpret_cast<int64_t*>(d_scal + 8);
            auto joined = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0),
                                                          JoinKey{lo_a, hi_a, b});
            size_t tmp2 = 0;
            GC_CUDA(c, cub::DeviceSelect::Unique(nullptr, tmp2, joined, c->canon.as<uint64_t>(), d_nsel, nnz,
                                                 c->stream));
            GC_TRY(ensure(c, c->cub_tmp, tmp2));
            tmp2 = c->cub_tmp.cap;
            GC_CUDA(c, cub::DeviceSelect::Unique(c->cub_tmp.p, tmp2, joined, c->canon.as<uint64_t>(), d_nsel, nnz,
                                                 c->stream));
            c->stats.lib_launches += 2;
            joined_done = true;
        } else {
            GC_LAUNCH(c, k_pack, grid_for(nnz), kThreads, 0, c->raw_u.as<int32_t>(), c->raw_v.as<int32_t>(), nnz, b,
                      sent, c->keys_a.as<uint64_t>());
            GC_TRY(radix_sort(c, c->keys_a.as<uint64_t>(), c->keys_b.as<uint64_t>(), nullptr, nullptr, nnz, 2 * b));
        }
        GC_TRY(ensure(c, c->canon, (size_t)nnz * 8));
        int64_t* d_nsel = reinterpret_cast<int64_t*>(d_scal + 8);
        if (!joined_done) {
            size_t tmp = 0;
            GC_CUDA(c, cub::DeviceSelect::Unique(nullptr, tmp, c->keys_b.as<uint64_t>(), c->canon.as<uint64_t>(),
                                                 d_nsel, nnz, c->stream));
            GC_TRY(ensure(c, c->cub_tmp, tmp));
            tmp = c->cub_tmp.cap;
            GC_CUDA(c, cub::DeviceSelect::Unique(c->cub_tmp.p, tmp, c->keys_b.as<uint64_t>(),
                                                 c->canon.as<uint64_t>(), d_nsel, nnz, c->stream));
            c->stats.lib_launches += 2;
        }
        GC_TRY(read_small(c, h, d_nsel, 8));
        GC_TRY(sync(c));
        int64_t nsel = h[0];
        if (nsel > 0) {
            GC_TRY(read_small(c, h + 1, c->canon.as<uint64_t>() + nsel - 1, 8));
            GC_TRY(sync(c));
            m = nsel - ((uint64_t)h[1] == sent ? 1 : 0);
        }
    }
    if (m >= ((int64_t)1 << 31) - 1) return fail(c, GC_ERR_RANGE, "gc_build_csr: m >= 2^31 (edge ids are int32)");
    c->m = m;

    // ---- a3: degrees
    GC_TRY(ensure(c, c->deg, (size_t)n * 4));
    GC_TRY(ensure(c, c->rank_of, (size_t)n * 4));
    GC_TRY(ensure(c, c->dag_ptr, (size_t)(n + 1) * 8));
    GC_TRY(ensure(c, c->in_ptr, (size_t)(n + 1) * 8));
    GC_TRY(ensure(c, c->dag_col, (size_t)m * 4 + 64));   // +64: 16-byte vector loads may read past a row end
    GC_TRY(ensure(c, c->dag_src, (size_t)m * 4));
    GC_TRY(ensure(c, c->dag_eid, (size_t)m * 4));
    GC_TRY(ensure(c, c->in_pos, (size_t)m * 4));
    GC_TRY(ensure(c, c->in_src, (size_t)m * 4));
    GC_TRY(ensure(c, c->in_dst, (size_t)m * 4));
    GC_TRY(ensure(c, c->vals_a, (size_t)(m > n ? m : n) * 4));
    GC_TRY(ensure(c, c->vals_b, (size_t)(m > n ? m : n) * 4));
    GC_TRY(ensure(c, c->keys_a, (size_t)(m > n ? m : n) * 8));
    GC_TRY(ensure(c, c->keys_b, (size_t)(m > n ? m : n) * 8));
    GC_CUDA(c, cudaMemsetAsync(c->deg.p, 0, (size_t)n * 4, c->stream));
    if (m > 0) {
        int32_t* first = c->vals_a.as<int32_t>();        // n entries each; zero = no lo run
        int32_t* last = c->vals_b.as<int32_t>();
        GC_CUDA(c, cudaMemsetAsync(first, 0, (size_t)n * 4, c->stream));
        GC_CUDA(c, cudaMemsetAsync(last, 0, (size_t)n * 4, c->stream));
        GC_LAUNCH(c, k_degrees, grid_for(m), kThreads, 0, c->canon.as<uint64_t>(), m, b, c->deg.as<int32_t>(),
                  first, last);
        GC_LAUNCH(c, k_degrees_lo, grid_for(n), kThreads, 0, first, last, n, c->deg.as<int32_t>());
    }

    // ---- a4: rank = sorted position of (deg, id); relabel + orient
    if (n > 0) {
        // sort on the degree's bits only (max degree read back first)
        uint32_t* vk = reinterpret_cast<uint32_t*>(c->keys_a.p);
        uint32_t* vk_out = vk + n;
        int32_t* ids = c->vals_a.as<int32_t>();
        int32_t* ids_out = c->vals_b.as<int32_t>();
        int* d_maxdeg = d_scal + 4;
        GC_CUDA(c, cudaMemsetAsync(d_maxdeg, 0, sizeof(int), c->stream));
        GC_LAUNCH(c, k_vkeys, grid_for(n), kThreads, 0, c->deg.as<int32_t>(), n, vk, ids, d_maxdeg);
        GC_TRY(read_small(c, h, d_maxdeg, sizeof(int)));
        GC_TRY(sync(c));
        const int dbits = std::max(1, ceil_log2_u64((uint64_t)reinterpret_cast<int*>(h)[0] + 1));
        size_t tmp = 0;
        GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, vk, vk_out, ids, ids_out, n, 0, dbits, c->stream));
        GC_TRY(ensure(c, c->cub_tmp, tmp));
        tmp = c->cub_tmp.cap;
        GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, vk, vk_out, ids, ids_out, n, 0, dbits,
                                                   c->stream));
        c->stats.lib_launches += 2 + (dbits + 7) / 8;
        GC_LAUNCH(c, k_rank_scatter, grid_for(n), kThreads, 0, ids_out, n, c->rank_of.as<int32_t>());
    }
    if (part) {
        GC_TRY(part_orient(c, n, b, m));
        GC_TRY(part_inlists(c, n, b, m));
    }
    if (m > 0 && !part) {
        GC_LAUNCH(c, k_orient, grid_for(m), kThreads, 0, c->canon.as<uint64_t>(), m, b, c->rank_of.as<int32_t>(),
                  c->keys_a.as<uint64_t>(), c->vals_a.as<int32_t>());
        GC_TRY(radix_sort(c, c->keys_a.as<uint64_t>(), c->keys_b.as<uint64_t>(), c->vals_a.as<int32_t>(),
                          c->dag_eid.as<int32_t>(), m, 2 * b));
    }
    if (!part) {
        // split the sorted keys into (dag_col, dag_src) and the row bounds in one pass;
        // keys_a is free after the sort: first / last there, row lengths in vals_a
        int32_t* first = reinterpret_cast<int32_t*>(c->keys_a.p);
        int32_t* last = first + n;
        GC_CUDA(c, cudaMemsetAsync(first, 0, (size_t)n * 8, c->stream));
        if (m > 0)
            GC_LAUNCH(c, k_split_keys_bounds, grid_for(m), kThreads, 0, c->keys_b.as<uint64_t>(), m, b,
                      c->dag_col.as<int32_t>(), c->dag_src.as<int32_t>(), first, last);
        GC_TRY(ensure(c, c->tmp_a, (size_t)(n + 1) * 8));
        GC_TRY(ptr_from_bounds(c, first, last, n, c->tmp_a.as<int64_t>(), c->dag_ptr.as<int64_t>()));
    }
    // in-lists: sort (head, tail) with the DAG position as payload
    if (part) {
        // built by part_inlists
    } else if (m > 0) {
        // DAG order is sorted by (tail, head): a stable sort on the head alone
        // (b-bit keys, 32-bit) groups in-edges by head with tails ascending.
        uint64_t* pv = c->keys_a.as<uint64_t>();          // free after the orientation sort
        uint64_t* pv_out = c->keys_b.as<uint64_t>();
        GC_LAUNCH(c, k_pos_tail, grid_for(m), kThreads, 0, c->dag_src.as<int32_t>(), m, pv);
        size_t tmp = 0;
        const uint32_t* hk = reinterpret_cast<const uint32_t*>(c->dag_col.p);
        uint32_t* hk_out = reinterpret_cast<uint32_t*>(c->in_dst.p);
        GC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, hk, hk_out, pv, pv_out, m, 0, b, c->stream));
        GC_TRY(ensure(c, c->cub_tmp, tmp));
        tmp = c->cub_tmp.cap;
        GC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, hk, hk_out, pv, pv_out, m, 0, b, c->stream));
        c->stats.lib_launches += 2 + (b + 7) / 8;
        int32_t* first = reinterpret_cast<int32_t*>(c->keys_a.p);   // pv (keys_a) consumed by the sort
        int32_t* last = first + n;
        GC_CUDA(c, cudaMemsetAsync(first, 0, (size_t)n * 8, c->stream));
        GC_LAUNCH(c, k_split_pos_tail_bounds, grid_for(m), kThreads, 0, pv_out, c->in_dst.as<int32_t>(), m,
                  c->in_pos.as<int32_t>(), c->in_src.as<int32_t>(), first, last);
        GC_TRY(ensure(c, c->tmp_a, (size_t)(n + 1) * 8));
        GC_TRY(ptr_from_bounds(c, first, last, n, c->tmp_a.as<int64_t>(), c->in_ptr.as<int64_t>()));
    } else {
        GC_TRY(csr_ptr_from_sorted(c, c->in_dst.as<int32_t>(), m, n, c->in_ptr.as<int64_t>()));
    }

    // ---- work-model statistics (one reduction over vertices)
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 512);
    GC_CUDA(c, cudaMemsetAsync(acc, 0, 13 * 8, c->stream));
    if (n > 0)
        GC_LAUNCH(c, k_graph_stats, grid_for(n), kThreads, 0, c->dag_ptr.as<int64_t>(), c->in_ptr.as<int64_t>(),
                  c->deg.as<int32_t>(), c->dag_col.as<int32_t>(), n, acc);
    GC_TRY(read_small(c, h, acc, 13 * 8));
    GC_TRY(sync(c));
    c->stats.n = n;
    c->stats.m = m;
    c->stats.wedges = h[0];
    c->stats.q_out = h[1];
    c->stats.q_in = h[2];
    c->stats.max_out_degree = h[3];
    c->stats.max_degree = h[4];
    for (int k = 0; k < 8; ++k) c->stats.aux[k] = h[5 + k];
    return GC_OK;
}

int get_edges(gc_ctx* c, int32_t* u_out, int32_t* v_out) {
    const int64_t m = c->m;
    if (m == 0) return GC_OK;
    GC_TRY(ensure(c, c->vals_a, (size_t)m * 4));
    GC_TRY(ensure(c, c->vals_b, (size_t)m * 4));
    GC_LAUNCH(c, k_unpack_canon, grid_for(m), kThreads, 0, c->canon.as<uint64_t>(), m, c->bits,
              c->vals_a.as<int32_t>(), c->vals_b.as<int32_t>());
    GC_TRY(copy_out(c, u_out, c->vals_a.p, (size_t)m * 4));
    GC_TRY(copy_out(c, v_out, c->vals_b.p, (size_t)m * 4));
    GC_TRY(sync(c));
    return GC_OK;
}

}  // namespace gcx

extern "C" int gc_get_edges(gc_ctx* c, int32_t* u_out, int32_t* v_out) {
    if (!c) return GC_ERR_INVALID;
    if (c->poisoned) return GC_ERR_STATE;
    if (c->state < 2) return gcx::fail(c, GC_ERR_STATE, "gc_get_edges before gc_build_csr");
    if (c->m > 0 && (!u_out || !v_out)) return gcx::fail(c, GC_ERR_INVALID, "gc_get_edges: NULL output");
    cudaSetDevice(c->device);
    return gcx::get_edges(c, u_out, v_out);
}
