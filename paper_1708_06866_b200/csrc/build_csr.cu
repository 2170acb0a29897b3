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
#include <cub/device/device_segmented_sort.cuh>
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

// ---- counting-sort build (GC_OPT_BUILD = 1): bucket by one endpoint with
// a histogram, an exclusive scan and an atomic scatter, then sort each
// bucket (CUB DeviceSegmentedSort: buckets are short -- a row of the graph
// -- so each is sorted in registers / shared memory in one pass instead of
// 3-6 global radix passes over every element).  Slots inside a bucket come
// from atomic decrements, so the order before the segmented sort is
// arbitrary; the sort makes the result deterministic (every rank of a
// communicator builds the same CSR).

// raw pairs per low endpoint (self loops dropped)
__global__ void k_count_lo(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t nnz,
                           unsigned long long* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = (uint32_t)__ldg(u + i), c = (uint32_t)__ldg(v + i);
        if (a != c) atomicAdd(cnt + min(a, c), 1ULL);
    }
}

// key (lo << b) | hi into lo's bucket (slots taken from the bucket's end)
__global__ void k_scatter_lo(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t nnz, int b,
                             const int64_t* __restrict__ ptr, unsigned long long* __restrict__ cnt,
                             uint64_t* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = (uint32_t)__ldg(u + i), c = (uint32_t)__ldg(v + i);
        if (a == c) continue;
        const uint32_t lo = min(a, c), hi = max(a, c);
        const int64_t slot = ptr[lo] + (int64_t)atomicAdd(cnt + lo, ~0ULL) - 1;   // atomic decrement
        keys[slot] = ((uint64_t)lo << b) | hi;
    }
}

// out-degree of every tail (lower rank) of the canonical edges
__global__ void k_orient_count(const uint64_t* __restrict__ canon, int64_t m, int b,
                               const int32_t* __restrict__ rank_of, unsigned long long* __restrict__ cnt) {
    const uint64_t mask = (1ULL << b) - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = canon[e];
        const uint32_t ra = (uint32_t)__ldg(rank_of + (k >> b)), rb = (uint32_t)__ldg(rank_of + (k & mask));
        atomicAdd(cnt + min(ra, rb), 1ULL);
    }
}

// (head << 32) | canonical id into the tail's row; the tail goes to dag_src
__global__ void k_orient_scatter(const uint64_t* __restrict__ canon, int64_t m, int b,
                                 const int32_t* __restrict__ rank_of, const int64_t* __restrict__ ptr,
                                 unsigned long long* __restrict__ cnt, uint64_t* __restrict__ rows,
                                 int32_t* __restrict__ dag_src) {
    const uint64_t mask = (1ULL << b) - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = canon[e];
        const uint32_t ra = (uint32_t)__ldg(rank_of + (k >> b)), rb = (uint32_t)__ldg(rank_of + (k & mask));
        const uint32_t t = min(ra, rb), h = max(ra, rb);
        const int64_t slot = ptr[t] + (int64_t)atomicAdd(cnt + t, ~0ULL) - 1;
        rows[slot] = ((uint64_t)h << 32) | (uint32_t)e;
        dag_src[slot] = (int32_t)t;
    }
}

__global__ void k_split_rows(const uint64_t* __restrict__ rows, int64_t m, int32_t* __restrict__ col,
                             int32_t* __restrict__ eid) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x = rows[p];
        col[p] = (int32_t)(x >> 32);
        eid[p] = (int32_t)(uint32_t)x;
    }
}

// in-degree of every head; lanes with the same head add once (a hub is the
// head of many short rows that share a warp)
__global__ void k_count_head(const int32_t* __restrict__ dag_col, int64_t m, unsigned long long* __restrict__ cnt) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t h = dag_col[p];
        const unsigned grp = __match_any_sync(__activemask(), h);
        if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(cnt + h, (unsigned long long)__popc(grp));
    }
}

// DAG position p into its head's in-list segment
__global__ void k_in_scatter(const int32_t* __restrict__ dag_col, int64_t m, const int64_t* __restrict__ ptr,
                             unsigned long long* __restrict__ cnt, uint32_t* __restrict__ pos) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t h = dag_col[p];
        const int64_t slot = ptr[h] + (int64_t)atomicAdd(cnt + h, ~0ULL) - 1;
        pos[slot] = (uint32_t)p;
    }
}

// in-list entry i (DAG position p, sorted per head): tail and head
__global__ void k_in_fill(const int32_t* __restrict__ in_pos, int64_t m, const int32_t* __restrict__ dag_src,
                          const int32_t* __restrict__ dag_col, int32_t* __restrict__ in_src,
                          int32_t* __restrict__ in_dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = in_pos[i];
        in_src[i] = dag_src[p];
        in_dst[i] = dag_col[p];
    }
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

// ptr = exclusive scan of the n + 1 counts (cnt[n] = 0)
static int scan_counts(gc_ctx* c, const unsigned long long* cnt, int64_t n, int64_t* ptr) {
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, ptr, n + 1, c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, cnt, ptr, n + 1, c->stream));
    c->stats.lib_launches += 2;
    return GC_OK;
}

// sort every segment [ptr[x], ptr[x+1]) of keys_in into keys_out
template <class K>
static int seg_sort(gc_ctx* c, const K* keys_in, K* keys_out, int64_t N, int64_t n, const int64_t* ptr) {
    if (N <= 0) return GC_OK;
    size_t tmp = 0;
    GC_CUDA(c, cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, keys_in, keys_out, (int)N, (int)n, ptr, ptr + 1,
                                                  c->stream));
    GC_TRY(ensure(c, c->cub_tmp, tmp));
    tmp = c->cub_tmp.cap;
    GC_CUDA(c, cub::DeviceSegmentedSort::SortKeys(c->cub_tmp.p, tmp, keys_in, keys_out, (int)N, (int)n, ptr, ptr + 1,
                                                  c->stream));
    c->stats.lib_launches += 4;   // partition + small / medium + large segment kernels (estimate)
    return GC_OK;
}

int build_csr(gc_ctx* c) {
    const int64_t nnz = c->nnz;
    c->n = 0;
    c->m = 0;
    c->bits = 1;
    c->build_v2_done = false;
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
    const uint64_t mask = (1ULL << b) - 1;

    // ---- a2: pack, sort, unique
    int64_t m = 0;
    if (nnz > 0) {
        GC_TRY(ensure(c, c->keys_a, (size_t)nnz * 8));
        GC_TRY(ensure(c, c->keys_b, (size_t)nnz * 8));
        const uint64_t sent = (2 * b >= 64) ? ~0ULL : ((1ULL << (2 * b)) - 1);
        bool joined_done = false;
        if (c->build_mode == 1 && b <= 31 && n <= ((int64_t)1 << 31) - 2) {
            // bucket the raw pairs by their low endpoint, sort each bucket, unique
            GC_TRY(ensure(c, c->tmp_a, (size_t)(n + 1) * 8));
            GC_TRY(ensure(c, c->tmp_b, (size_t)(n + 1) * 8));
            unsigned long long* cnt = c->tmp_a.as<unsigned long long>();
            int64_t* ptr = c->tmp_b.as<int64_t>();
            GC_CUDA(c, cudaMemsetAsync(cnt, 0, (size_t)(n + 1) * 8, c->stream));
            GC_LAUNCH(c, k_count_lo, grid_for(nnz), kThreads, 0, c->raw_u.as<int32_t>(), c->raw_v.as<int32_t>(), nnz,
                      cnt);
            GC_TRY(scan_counts(c, cnt, n, ptr));
            GC_TRY(read_small(c, h, ptr + n, 8));
            GC_TRY(sync(c));
            const int64_t nv = h[0];                        // pairs that are no self loop
            if (nv > 0) {
                GC_LAUNCH(c, k_scatter_lo, grid_for(nnz), kThreads, 0, c->raw_u.as<int32_t>(), c->raw_v.as<int32_t>(),
                          nnz, b, ptr, cnt, c->keys_a.as<uint64_t>());
                GC_TRY(seg_sort<uint64_t>(c, c->keys_a.as<uint64_t>(), c->keys_b.as<uint64_t>(), nv, n, ptr));
                GC_TRY(ensure(c, c->canon, (size_t)nnz * 8));
                int64_t* d_nsel = reinterpret_cast<int64_t*>(d_scal + 8);
                size_t tmp2 = 0;
                GC_CUDA(c, cub::DeviceSelect::Unique(nullptr, tmp2, c->keys_b.as<uint64_t>(), c->canon.as<uint64_t>(),
                                                     d_nsel, nv, c->stream));
                GC_TRY(ensure(c, c->cub_tmp, tmp2));
                tmp2 = c->cub_tmp.cap;
                GC_CUDA(c, cub::DeviceSelect::Unique(c->cub_tmp.p, tmp2, c->keys_b.as<uint64_t>(),
                                                     c->canon.as<uint64_t>(), d_nsel, nv, c->stream));
                c->stats.lib_launches += 2;
                GC_TRY(read_small(c, h, d_nsel, 8));
                GC_TRY(sync(c));
                m = h[0];
            }
            joined_done = true;
            c->build_v2_done = true;
        } else if (GC_SPLIT_SORT1 && b <= 31) {
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
        if (c->build_v2_done) {
            // m known, no self-loop sentinel in the list
        } else if (!joined_done) {
            size_t tmp = 0;
            GC_CUDA(c, cub::DeviceSelect::Unique(nullptr, tmp, c->keys_b.as<uint64_t>(), c->canon.as<uint64_t>(),
                                                 d_nsel, nnz, c->stream));
            GC_TRY(ensure(c, c->cub_tmp, tmp));
            tmp = c->cub_tmp.cap;
            GC_CUDA(c, cub::DeviceSelect::Unique(c->cub_tmp.p, tmp, c->keys_b.as<uint64_t>(),
                                                 c->canon.as<uint64_t>(), d_nsel, nnz, c->stream));
            c->stats.lib_launches += 2;
        }
        if (!c->build_v2_done) {
        GC_TRY(read_small(c, h, d_nsel, 8));
        GC_TRY(sync(c));
        int64_t nsel = h[0];
        if (nsel > 0) {
            GC_TRY(read_small(c, h + 1, c->canon.as<uint64_t>() + nsel - 1, 8));
            GC_TRY(sync(c));
            m = nsel - ((uint64_t)h[1] == sent ? 1 : 0);
        }
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
    if (c->build_mode == 1) {
        // DAG rows: out-degree histogram, scan, scatter (head, id) into the
        // tail's row, sort each row by head.  In-lists: in-degree histogram,
        // scan, scatter the DAG position into the head's segment, sort each
        // segment (DAG positions ascend with the tail).
        GC_TRY(ensure(c, c->tmp_a, (size_t)(n + 1) * 8));
        unsigned long long* cnt = c->tmp_a.as<unsigned long long>();
        int64_t* dptr = c->dag_ptr.as<int64_t>();
        int64_t* iptr = c->in_ptr.as<int64_t>();
        GC_CUDA(c, cudaMemsetAsync(cnt, 0, (size_t)(n + 1) * 8, c->stream));
        if (m > 0)
            GC_LAUNCH(c, k_orient_count, grid_for(m), kThreads, 0, c->canon.as<uint64_t>(), m, b,
                      c->rank_of.as<int32_t>(), cnt);
        GC_TRY(scan_counts(c, cnt, n, dptr));
        if (m > 0) {
            GC_LAUNCH(c, k_orient_scatter, grid_for(m), kThreads, 0, c->canon.as<uint64_t>(), m, b,
                      c->rank_of.as<int32_t>(), dptr, cnt, c->keys_a.as<uint64_t>(), c->dag_src.as<int32_t>());
            GC_TRY(seg_sort<uint64_t>(c, c->keys_a.as<uint64_t>(), c->keys_b.as<uint64_t>(), m, n, dptr));
            GC_LAUNCH(c, k_split_rows, grid_for(m), kThreads, 0, c->keys_b.as<uint64_t>(), m, c->dag_col.as<int32_t>(),
                      c->dag_eid.as<int32_t>());
        }
        GC_CUDA(c, cudaMemsetAsync(cnt, 0, (size_t)(n + 1) * 8, c->stream));
        if (m > 0) GC_LAUNCH(c, k_count_head, grid_for(m), kThreads, 0, c->dag_col.as<int32_t>(), m, cnt);
        GC_TRY(scan_counts(c, cnt, n, iptr));
        if (m > 0) {
            uint32_t* pos = reinterpret_cast<uint32_t*>(c->keys_a.p);
            GC_LAUNCH(c, k_in_scatter, grid_for(m), kThreads, 0, c->dag_col.as<int32_t>(), m, iptr, cnt, pos);
            GC_TRY(seg_sort<uint32_t>(c, pos, reinterpret_cast<uint32_t*>(c->in_pos.p), m, n, iptr));
            GC_LAUNCH(c, k_in_fill, grid_for(m), kThreads, 0, c->in_pos.as<int32_t>(), m, c->dag_src.as<int32_t>(),
                      c->dag_col.as<int32_t>(), c->in_src.as<int32_t>(), c->in_dst.as<int32_t>());
        }
    }
    if (m > 0 && c->build_mode != 1) {
        GC_LAUNCH(c, k_orient, grid_for(m), kThreads, 0, c->canon.as<uint64_t>(), m, b, c->rank_of.as<int32_t>(),
                  c->keys_a.as<uint64_t>(), c->vals_a.as<int32_t>());
        GC_TRY(radix_sort(c, c->keys_a.as<uint64_t>(), c->keys_b.as<uint64_t>(), c->vals_a.as<int32_t>(),
                          c->dag_eid.as<int32_t>(), m, 2 * b));
    }
    if (c->build_mode != 1) {
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
    if (c->build_mode == 1) {
        // built above
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
