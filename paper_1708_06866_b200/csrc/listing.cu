// listing.cu — triangle listing: Alg. 1's triangle
// records {i, x, y} (P:187-200 [Triangle counting]: "the triangles ... can be
// enumerated"), here as vertex-id triples.
//
// Every triangle u < v < w (ranks) is listed once, from its DAG edge u -> v:
// the common out-neighbours w of u and v (N+(u) ∩ N+(v), both rows sorted by
// rank and short, d+ <= sqrt(2m)).  One warp per DAG edge walks the shorter
// row and binary-searches the longer; hits are appended through a warp-
// aggregated atomic cursor.  Output triples hold ORIGINAL ids sorted
// ascending within the triple; the order of the triples is unspecified.
#include "gc_internal.cuh"

namespace gcx {

namespace {

__global__ void k_id_of_rank(const int32_t* __restrict__ rank_of, int64_t n, int32_t* __restrict__ id_of) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
        id_of[rank_of[x]] = (int32_t)x;
}

__device__ __forceinline__ int64_t lb_i32(const int32_t* __restrict__ a, int64_t lo, int64_t hi, int32_t x) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_list(const int32_t* __restrict__ dag_src, const int32_t* __restrict__ dag_col,
                                              const int64_t* __restrict__ dag_ptr, const int32_t* __restrict__ id_of,
                                              int64_t m, int32_t* __restrict__ out, unsigned long long* __restrict__ cursor,
                                              int64_t capacity) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < m; p += nw) {
        const int u = dag_src[p], v = dag_col[p];
        int64_t a0 = p + 1, a1 = dag_ptr[u + 1];        // N+(u) past v (entries rank above v)
        int64_t b0 = dag_ptr[v], b1 = dag_ptr[v + 1];   // N+(v)
        if (a1 - a0 > b1 - b0) {
            int64_t t0 = a0, t1 = a1;
            a0 = b0; a1 = b1; b0 = t0; b1 = t1;
        }
        for (int64_t base = a0; base < a1; base += 32) {
            const int64_t i = base + lane;
            int32_t w = -1;
            bool hit = false;
            if (i < a1) {
                w = __ldg(dag_col + i);
                const int64_t j = lb_i32(dag_col, b0, b1, w);
                hit = j < b1 && __ldg(dag_col + j) == w;
            }
            const unsigned hm = __ballot_sync(0xffffffffu, hit);
            if (!hm) continue;
            unsigned long long slot = 0;
            if (lane == 0) slot = atomicAdd(cursor, (unsigned long long)__popc(hm));
            slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(hm & ((1u << lane) - 1));
            if (hit && (int64_t)slot < capacity) {
                int32_t x = id_of[u], y = id_of[v], z = id_of[w];
                // sort the three ids ascending
                if (x > y) { int32_t t = x; x = y; y = t; }
                if (y > z) { int32_t t = y; y = z; z = t; }
                if (x > y) { int32_t t = x; x = y; y = t; }
                out[3 * slot] = x;
                out[3 * slot + 1] = y;
                out[3 * slot + 2] = z;
            }
        }
    }
}

}  // namespace

int list_triangles(gc_ctx* c, int32_t* tri_out, int64_t capacity, int64_t* count) {
    uint64_t T = 0;
    GC_TRY(triangle_count(c, &T));          // exact size first (a TC pass)
    *count = (int64_t)T;
    if ((int64_t)T > capacity) return fail(c, GC_ERR_RANGE, "gc_list_triangles: capacity below the triangle count");
    if (T == 0) return GC_OK;
    const int64_t n = c->n, m = c->m;
    GC_TRY(ensure(c, c->id_of, (size_t)n * 4));
    GC_TRY(ensure(c, c->list_out, (size_t)T * 12));
    GC_TRY(ensure(c, c->scal, 1024));
    unsigned long long* cursor = reinterpret_cast<unsigned long long*>(c->scal.as<char>() + 296);
    GC_CUDA(c, cudaMemsetAsync(cursor, 0, 8, c->stream));
    GC_LAUNCH(c, k_id_of_rank, grid_for(n), kThreads, 0, c->rank_of.as<int32_t>(), n, c->id_of.as<int32_t>());
    GC_LAUNCH(c, k_list, grid_for(m * 32), kThreads, 0, c->dag_src.as<int32_t>(), c->dag_col.as<int32_t>(),
              c->dag_ptr.as<int64_t>(), c->id_of.as<int32_t>(), m, c->list_out.as<int32_t>(), cursor, (int64_t)T);
    GC_TRY(copy_out(c, tri_out, c->list_out.p, (size_t)T * 12));
    GC_TRY(sync(c));
    return GC_OK;
}

}  // namespace gcx

extern "C" int gc_list_triangles(gc_ctx* c, int32_t* tri_out, int64_t capacity, int64_t* count) {
    if (!c) return GC_ERR_INVALID;
    if (c->poisoned) return GC_ERR_STATE;
    if (c->state < 2) return gcx::fail(c, GC_ERR_STATE, "gc_list_triangles before gc_build_csr");
    if (!count || capacity < 0 || (capacity > 0 && !tri_out))
        return gcx::fail(c, GC_ERR_INVALID, "gc_list_triangles: bad arguments");
    cudaSetDevice(c->device);
    return gcx::list_triangles(c, tri_out, capacity, count);
}
