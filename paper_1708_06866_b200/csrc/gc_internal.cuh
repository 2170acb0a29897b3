// gc_internal.cuh — libgc internals: context, device buffers, error plumbing.
//
// Layout in HBM: every graph array lives in one
// gc_ctx and is reused across calls (grow-only, stream-ordered allocations
// from the CUDA memory pool), so a steady-state step allocates nothing.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "gc.h"

namespace gcx {

constexpr int kClasses = 5;   // intersection kernel classes: 0 lane, 1 warp, 2 block, 3 huge, 4 wide bitmap

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// Status plumbing ------------------------------------------------------------
#define GC_TRY(expr)                         \
    do {                                     \
        int _rc = (expr);                    \
        if (_rc != GC_OK) return _rc;        \
    } while (0)

#define GC_CUDA(ctx, expr)                                                         \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) return gcx::cuda_fail((ctx), _e, #expr, __FILE__, __LINE__); \
    } while (0)

// Every libgc kernel launch goes through this macro: it counts the launch
// (gc_stats.launches, the bench's "gpu_launches") and checks the launch.
#define GC_LAUNCH(ctx, kernel, grid, block, smem, ...)                                  \
    do {                                                                                \
        (ctx)->stats.launches++;                                                        \
        kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);                \
        cudaError_t _e = cudaGetLastError();                                            \
        if (_e != cudaSuccess) return gcx::cuda_fail((ctx), _e, #kernel, __FILE__, __LINE__); \
    } while (0)

#define GC_LAUNCH_S(ctx, strm, kernel, grid, block, smem, ...)                          \
    do {                                                                                \
        (ctx)->stats.launches++;                                                        \
        kernel<<<(grid), (block), (smem), (strm)>>>(__VA_ARGS__);                       \
        cudaError_t _e = cudaGetLastError();                                            \
        if (_e != cudaSuccess) return gcx::cuda_fail((ctx), _e, #kernel, __FILE__, __LINE__); \
    } while (0)

}  // namespace gcx

struct gc_ctx {
    int device = 0;
    cudaMemPool_t pool = nullptr;    // library-owned stream-ordered pool (release threshold: keep everything)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t side = nullptr;     // library-owned side stream (warp-task classes overlap the block kernels)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int overlap = 1;                 // GC_OPT_OVERLAP
    int launch_grid[5][2] = {};      // intersection kernels: occupancy grid per class and SUP (0: not yet set up)
    std::string err;
    bool poisoned = false;
    int state = 0;  // 0 created, 1 edges loaded, 2 graph built

    // options
    int force_class = -1;
    int build_part = -1;             // GC_OPT_BUILD_PART: -1 auto (partitioned build when parts > 1), 0 replicated, 1 partitioned
    int64_t task_chunk = 32768;
    int timing = 1;
    int block_bitmap = 1;
    int long_seg = 48;
    int block_batch = 32;
    int sup_skip = 0;
    int huge_max = 8192;   // class 3: largest d+ in the 16384-slot shared hash (GC_OPT_HUGE_MAX)

    // raw input (a1)
    gcx::Buf raw_u, raw_v;
    gcx::Buf stage_u, stage_v;       // gc_stage_edges: the next graph's raw list
    int64_t stage_nnz = -1;          // >= 0: a staged list waits for the next gc_build_csr
    cudaStream_t copy_s = nullptr;   // library-owned copy stream of gc_stage_edges (lazy)
    cudaEvent_t ev_staged = nullptr;
    cudaStream_t d2h_s = nullptr;    // library-owned read-back stream of gc_ktruss_analysis_async (lazy)
    cudaEvent_t ev_out_ready = nullptr, ev_d2h_done = nullptr;
    bool d2h_pending = false;        // out_tmp / out_tmp2 are being read back
    bool async_out = false;          // the running call delivers per-edge outputs asynchronously
    int64_t nnz = 0;

    // graph sizes
    int64_t n = 0, m = 0;
    int bits = 1;  // b: vertex id bits; keys pack (hi << b) | lo

    // canonical list (a2): uint64 key (min << b) | max, m entries
    gcx::Buf canon;
    // degrees (a3), rank relabelling (a4)
    gcx::Buf deg;       // int32[n]
    gcx::Buf rank_of;   // int32[n] old id -> rank (new id)
    // oriented DAG in rank space (a4): row x = N+(x) ascending
    gcx::Buf dag_ptr;   // int64[n+1]
    gcx::Buf dag_col;   // int32[m]
    gcx::Buf dag_src;   // int32[m]
    gcx::Buf dag_eid;   // int32[m] canonical edge id of DAG position p
    // in-lists grouped by head v, ascending tail u (a4/a5)
    gcx::Buf in_ptr;    // int64[n+1]
    gcx::Buf in_pos;    // int32[m]  DAG position p of edge u->v
    gcx::Buf in_src;    // int32[m]  u
    gcx::Buf in_dst;    // int32[m]  v (head; in-list is sorted by (v, u))
    // intersection tasks (a5)
    gcx::Buf task_i0;   // int32 first in-list index of each task (tasks grouped by class)
    gcx::Buf task_i1;   // int32 one past the last in-list index of each task
    gcx::Buf in_cost;   // int64[m] exclusive cost prefix over the in-list
    gcx::Buf tmp_a, tmp_b;  // task construction scratch
    int64_t ntask[5] = {0, 0, 0, 0, 0};      // per intersection class (gcx::kClasses)
    int64_t task_off[6] = {0, 0, 0, 0, 0, 0};
    int64_t total_cost = 0;
    gcx::Buf task_pref;     // int64 exclusive cost prefix over the class-sorted tasks (multi-owner cut)
    int64_t cls_start[5] = {0, 0, 0, 0, 0}, cls_total[5] = {1, 1, 1, 1, 1};
    int task_parts = 1;     // number of owners the tasks were cut for
    bool tasks_ready = false;

    // scratch
    gcx::Buf keys_a, keys_b;    // uint64 sort buffers
    gcx::Buf vals_a, vals_b;    // int32 sort payloads
    gcx::Buf cub_tmp;
    gcx::Buf scal;              // small device scalars (counters, reductions)
    gcx::Buf sup;               // uint32[m] support in DAG-position order
    gcx::Buf uw16;              // uint16[m] (u,w)-role credits of the support pass (folded into sup)
    gcx::Buf out_tmp;           // staging for canonical-order outputs
    gcx::Buf out_tmp2;          // second staging buffer (fused analysis: support and mask)
    gcx::Buf id_of;             // int32[n] rank -> original id (triangle listing)
    gcx::Buf list_out;          // int32[3T] listed triangles

    // peeler (a8/a9)
    gcx::Buf sym_ptr;   // int64[n+1]
    gcx::Buf sym_col;   // int32[2m]
    gcx::Buf sym_eid;   // int32[2m] DAG position of the edge
    bool sym_ready = false;
    bool sym_dirty = true;  // rows were compacted (or never filled): refill before the next peel
    bool rows_live = false; // rows filled for the current peel call
    gcx::Buf live_len;  // int32[n] live entries at the front of each symmetric row
    gcx::Buf long_rows; // int32 rows longer than kLongRow (compacted block-wide)
    int nlong = 0;
    gcx::Buf batch_slot;   // int64 per-block next-batch slots of the block-class kernels
    gcx::Buf grp_keys, grp_vals, grp_starts, grp_flags, grp_light;   // grouped dense-core rounds
    // frontier size from which k_peel runs its 64-register build (diagnostics; default never: with two
    // searches in flight per lane the full-occupancy 32-register build wins at every frontier size)
    int64_t peel_big = getenv("GC_PEEL_BIG") ? atoll(getenv("GC_PEEL_BIG")) : INT64_MAX;
    int group_peel = 0;         // GC_OPT_GROUP_PEEL: frontier size from which a round groups its heavy edges (0: never)
    int group_heavy = 1024;     // GC_OPT_GROUP_HEAVY: shorter live row from which a frontier edge is grouped
    int sort_front = 1 << 20;   // GC_OPT_SORT_FRONT: frontiers of at least this many edges sorted by probed row (0: never)
    gcx::Buf alist;     // int32 live-edge list of the last compaction (level scans)
    int64_t alist_n = -1;       // -1: no list (scan every edge)
    int64_t m_alive_h = 0;      // live edges (host mirror)
    int64_t compact_at = 0;     // live edges at the last compaction
    int trace = getenv("GC_PEEL_TRACE") ? atoi(getenv("GC_PEEL_TRACE")) : 0;   // diagnostics: 1 a line per batch, 2 per round
    int compact_div = 5;        // compact when live edges fall to (v-1)/v, v = compact_div (GC_OPT_COMPACT; <= 1 never)
    bool decomp_running = false;   // a truss decomposition is peeling (compact_div applies; else at most 2)
    gcx::Buf alive;     // uint8[m] edge state: 0 removed, 1 alive, 2 / 3 in the frontier (peel.cu st_front)
    gcx::Buf front_a, front_b;  // int32[m] frontier lists
    gcx::Buf tau;       // int32[m]
    gcx::Buf xbits;     // uint32 removed-edge bitmap X of the round (partitioned peel, allgathered)
    gcx::Buf nbits;     // uint32 next-round bitmap (each owner sets bits in its slice)
    gcx::Buf zbits;     // uint32 zero-support edges of a level start (removed without enumeration)
    gcx::Buf dec_out, dec_in;   // partitioned peel (NCCL): decrements of other ranks' edges, sent / received
    gcx::Buf sup_parts; // uint32[P*m] per-virtual-rank supports (loopback partitions only)
    int peel_part = 0;  // 1: partitioned (bitmap) peeler even on one rank (GC_OPT_PEEL_PART)
    int work_stats = 0; // GC_OPT_WORK_STATS: count the k-truss byte model's terms while peeling
    gcx::Buf vdeg;      // int32[n] alive degree per vertex (rank space; work stats only)
    gcx::Buf zlist;     // int32[m] edges removed at a level scan with S = 0 (work stats only)

    // pinned host scratch
    void* hpin = nullptr;
    size_t hpin_cap = 0;
    void* hpin_dev = nullptr;        // hpin mapped into the device address space (read_small)

    // events
    cudaEvent_t ev[14] = {};   // 0-7 phases; 8-13 peel sub-phases (kernel / scan / compaction)
    cudaEvent_t pev[17] = {};  // loopback partitions: per virtual rank intersection time (created on first use)

    gc_stats stats = {};

    // multi-GPU
    int nranks = 1, rank = 0;
    int loop_parts = 0;       // > 0: loopback virtual ranks on this GPU
    void* nccl = nullptr;     // ncclComm_t
};

namespace gcx {

int cuda_fail(gc_ctx* c, cudaError_t e, const char* what, const char* file, int line);
int fail(gc_ctx* c, int code, const std::string& msg);
int ensure(gc_ctx* c, Buf& b, size_t bytes);
void release(gc_ctx* c, Buf& b);
int host_scratch(gc_ctx* c, size_t bytes);
int sync(gc_ctx* c);
// copy nbytes from device src to a caller pointer (host or device)
int copy_out(gc_ctx* c, void* dst, const void* src_dev, size_t nbytes);
int copy_in(gc_ctx* c, void* dst_dev, const void* src, size_t nbytes);
// per-edge output staged in out_tmp / out_tmp2 -> caller: on the context
// stream, or on the read-back stream when c->async_out is set
int copy_out_staged(gc_ctx* c, void* dst, const void* src_dev, size_t nbytes);
// the context stream waits for a pending asynchronous read-back (before out_tmp / out_tmp2 are rewritten)
int claim_out(gc_ctx* c);
// a few bytes device -> the page-locked scratch c->hpin, ordered on the
// context stream, without a copy engine
int read_small(gc_ctx* c, void* host_dst, const void* src_dev, size_t nbytes);
float elapsed(gc_ctx* c, int a, int b);
int record(gc_ctx* c, int i);

// build_csr.cu
int build_csr(gc_ctx* c);
// tc.cu
int prepare_tasks(gc_ctx* c);
int triangle_count(gc_ctx* c, uint64_t* out);
int support_dag(gc_ctx* c);   // fills c->sup (DAG order), all ranks combined
unsigned long long* support_hits(gc_ctx* c);   // this rank's triangle count of the last support pass
int scatter_canonical_u32(gc_ctx* c, const uint32_t* dag_vals, uint32_t* canon_out_dev);
int scatter_canonical_u8(gc_ctx* c, const uint8_t* dag_vals, uint8_t* canon_out_dev);
// peel.cu
int build_sym(gc_ctx* c);
int ktruss(gc_ctx* c, int32_t k, uint8_t* alive_out, int64_t* m_alive);
int ktruss_analysis(gc_ctx* c, int32_t k, uint64_t* triangles, uint32_t* support_out, uint8_t* alive_out,
                    int64_t* m_alive);
int truss_decomposition(gc_ctx* c, int32_t* tau_out, int32_t* kmax);
// listing.cu
int list_triangles(gc_ctx* c, int32_t* tri_out, int64_t capacity, int64_t* count);
// comm.cu
int nccl_get_unique_id(void* id);
int nccl_init(gc_ctx* c, const void* id, int nranks, int rank);
int nccl_destroy(gc_ctx* c);
int allreduce_u64(gc_ctx* c, uint64_t* dev, size_t count);
int allreduce_u32(gc_ctx* c, uint32_t* dev, size_t count);
int allreduce_min_u32(gc_ctx* c, uint32_t* dev, size_t count);
int allreduce_max_u32(gc_ctx* c, uint32_t* dev, size_t count);
int allgather_u32(gc_ctx* c, const uint32_t* send, uint32_t* recv, size_t count_per_rank);
int allgatherv_i32(gc_ctx* c, const int32_t* send, int32_t* recv, const int64_t* counts, const int64_t* offsets);

inline int ceil_log2_u64(uint64_t x) {  // bits needed to represent values < x (x >= 1)
    int b = 0;
    while ((1ULL << b) < x) ++b;
    return b;
}

constexpr int kThreads = 256;
#ifndef GC_GRID_CAP
#define GC_GRID_CAP (148 * 64)   // grid-stride kernels: blocks at most (C4 build 45.0 -> 44.3 ms, level scans -5 % against 148 x 16;
                                 // one block per 256 elements was slower: build 54 ms, scans 2.7x)
#endif
inline int grid_for(int64_t n, int threads = kThreads, int cap = GC_GRID_CAP) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

}  // namespace gcx
