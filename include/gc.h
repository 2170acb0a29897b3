/*
 * gc.h — C ABI of libgc: per-edge triangle support, triangle count and
 * k-truss on NVIDIA B200 (sm_100a).
 *
 * Method: Samsi et al., "Static Graph Challenge: Subgraph Isomorphism"
 * (arXiv 1708.06866).  Citations "P:<n>" are lines of PAPER.md, section in
 * brackets.  The operation contracts follow SURVEY.md §8(b); readings of
 * ambiguous passages are listed in DESIGN.md ("Readings").
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Return value: GC_OK (0) or a gc_status code.  On error the message is
 *    available from gc_last_error(ctx).  After GC_ERR_CUDA or GC_ERR_NCCL the
 *    context is poisoned: every later call except gc_last_error/gc_destroy
 *    returns GC_ERR_STATE; destroy it.
 *  - Vertex ids are 0-based int32 (the paper's files are 1-based, P:134-144;
 *    the shift belongs to the file reader, not to this library).
 *  - Pointers passed in or out may be host memory (pageable or pinned) or
 *    device memory of the context's GPU (CUDA unified addressing decides).
 *    Inputs are copied before the call returns; the caller keeps ownership
 *    of every buffer it passes.  Output buffers are caller-allocated with
 *    the sizes stated below.
 *  - Every call returns after its outputs are complete (the context stream
 *    is synchronised before return).
 *  - Call order: gc_create -> [gc_comm_init | gc_comm_init_loopback] ->
 *    gc_load_edges -> gc_build_csr -> any of gc_triangle_count,
 *    gc_edge_support, gc_ktruss, gc_ktruss_analysis, gc_truss_decomposition,
 *    gc_list_triangles, gc_get_edges, any number of times.  A call out of
 *    order returns GC_ERR_STATE.
 *    gc_load_edges invalidates the built graph.
 *  - Edge ids: the canonical edge list is the set of undirected edges
 *    {min(u,v), max(u,v)} with u != v, sorted lexicographically; edge id =
 *    position in it.  Every per-edge output (support, mask, trussness) is in
 *    this order; gc_get_edges exports it.
 *  - Multi-GPU (after gc_comm_init): SPMD.  Every rank makes the same calls
 *    with the same full edge list; every call is collective; results are
 *    identical on all ranks.
 *  - A context is not thread-safe; distinct contexts are independent.
 */
#ifndef GC_H_
#define GC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gc_ctx gc_ctx;   /* opaque; one per (process, GPU) */

typedef enum gc_status {
    GC_OK = 0,
    GC_ERR_INVALID = 1,   /* bad argument (NULL pointer, negative id, k < 2, ...) */
    GC_ERR_STATE = 2,     /* call out of order, or context poisoned */
    GC_ERR_RANGE = 3,     /* graph exceeds index widths (m >= 2^31, n > 2^31) */
    GC_ERR_OOM = 4,       /* device allocation failed */
    GC_ERR_CUDA = 5,      /* CUDA runtime / kernel error (context poisoned) */
    GC_ERR_NCCL = 6       /* NCCL error or NCCL unavailable (context poisoned) */
} gc_status;

/* Create a context on CUDA device `device`.  cuda_stream: a cudaStream_t of
 * that device on which all work is queued, or NULL for a library-owned
 * stream.  *out receives the context. */
int gc_create(gc_ctx** out, int device, void* cuda_stream);

/* Free every device and host resource of ctx (NULL is a no-op). */
int gc_destroy(gc_ctx* ctx);

/* Message for the last error on ctx ("" if none).  Valid until the next
 * call on ctx.  ctx may be NULL (messages of gc_create failures). */
const char* gc_last_error(const gc_ctx* ctx);

/* ------------------------------------------------------------ multi-GPU --
 * NCCL over NVLink (libnccl.so.2 is resolved at run time with dlopen; the
 * process's already-loaded NCCL, e.g. PyTorch's, is reused).
 * gc_nccl_unique_id: rank 0 writes a 128-byte ncclUniqueId to id_out, which
 * the caller broadcasts (e.g. torch.distributed) to every rank.
 * gc_comm_init: join the communicator of nranks ranks as `rank`.  From then
 * on gc_triangle_count / gc_edge_support split their work into nranks
 * balanced 1D ranges of the oriented edge set and combine partial results
 * with ncclAllReduce; the k-truss peeler exchanges each round's removed-edge
 * bitmap with ncclAllGather.  Must precede gc_load_edges. */
int gc_nccl_unique_id(void* id_out /* 128 bytes */);
int gc_comm_init(gc_ctx* ctx, const void* nccl_unique_id, int nranks, int rank);

/* Host-only (no GPU, no context): the 1D work partition every rank computes
 * identically.  cost_prefix: len+1 int64 values, the
 * exclusive prefix sum of non-negative per-item costs (cost_prefix[len] =
 * total).  Item i belongs to owner min(nparts - 1,
 * floor(cost_prefix[i] * nparts / total)) (trailing zero-cost items go to the
 * last owner).
 * bounds_out[r] = first item of owner r (nondecreasing), bounds_out[nparts] =
 * len; owner r holds [bounds_out[r], bounds_out[r+1]).  The intersection
 * kernels apply the same rule to their task list.  Errors: NULL pointers,
 * len < 0, nparts < 1 -> GC_ERR_INVALID. */
int gc_partition_bounds(const int64_t* cost_prefix, int64_t len, int nparts, int64_t* bounds_out);

/* Testing aid for the partitioned path on ONE GPU: nparts virtual ranks run
 * one after another in this process and their partial results are combined
 * by device sums instead of NCCL.  Results must equal nparts = 1. */
int gc_comm_init_loopback(gc_ctx* ctx, int nparts);

/* ---------------------------------------------------------------- input --
 * gc_load_edges (north star "gc_load_edges(u,v,nnz)"; P:131-144 [Data
 * Sets]: edges as vectors u, v of vertex ids).
 * u, v: nnz int32 vertex ids each, raw directed pairs in any order; may
 * contain self loops, duplicates and both orientations (normalised by
 * gc_build_csr).  nnz >= 0.  n (vertex count) = max id + 1, 0 if
 * nnz == 0.  Errors: NULL with nnz > 0 -> GC_ERR_INVALID; a negative id is
 * reported by gc_build_csr. */
int gc_load_edges(gc_ctx* ctx, const int32_t* u, const int32_t* v, int64_t nnz);

/* gc_stage_edges: the load step (a1) of the NEXT graph, overlapped with work
 * on the current one.  Enqueues the copy of u, v (same meaning and checks
 * as gc_load_edges) on a library copy stream and returns at once; the
 * current edge list, CSR and results stay valid and usable.  The next
 * gc_build_csr waits for the copy and builds from the staged list.  A second
 * gc_stage_edges first waits for the pending copy and then replaces it;
 * gc_load_edges waits for and discards it.
 * Ownership: the caller keeps u, v and must leave them unchanged until that
 * gc_build_csr returns.  Page-locked host memory (or device memory) gives a
 * copy that overlaps the kernels; pageable host memory is accepted but the
 * driver copies it before returning.  Errors: as gc_load_edges; copy
 * failures are reported here or by the gc_build_csr that consumes it. */
int gc_stage_edges(gc_ctx* ctx, const int32_t* u, const int32_t* v, int64_t nnz);

/* gc_build_csr (north star): on the GPU, drop self loops, fold both
 * orientations and duplicates, sort into the canonical list;
 * compute degrees ("d = sum(E)"); rank vertices by (degree, id) and
 * orient every edge from lower to higher rank (the L/U split of P:234 after
 * relabelling by rank), and build the oriented CSR plus the per-edge work
 * table of the intersection kernels.
 * Errors: negative id -> GC_ERR_INVALID; canonical m >= 2^31 or
 * max id >= 2^31 - 1 -> GC_ERR_RANGE. */
int gc_build_csr(gc_ctx* ctx);

/* Graph sizes after gc_build_csr.  m = undirected, deduplicated,
 * self-loop-free edge count (the "number of edges" of P:319-320). */
int gc_num_vertices(const gc_ctx* ctx, int64_t* n);
int gc_num_edges(const gc_ctx* ctx, int64_t* m);

/* Canonical edge list: u_out[i] < v_out[i], lexicographic; m entries each. */
int gc_get_edges(gc_ctx* ctx, int32_t* u_out, int32_t* v_out);

/* --------------------------------------------------------------- kernels --
 * gc_triangle_count (north star; P:157-160 [Triangle counting]: "a set of
 * three mutually adjacent vertices"; Alg. 1-3).  *count = number
 * of triangles, each counted once.  64-bit. */
int gc_triangle_count(gc_ctx* ctx, uint64_t* count);

/* gc_edge_support (north star "per-edge triangle support"; P:283-288
 * [k-Truss]: support of an edge = overlap of its endpoints' neighbourhoods,
 * the count of 2s in its row of EA).  support_out[i] = |N(u_i) ∩ N(v_i)| for
 * canonical edge i; m uint32 entries.  Sum over edges = 3 * triangles. */
int gc_edge_support(gc_ctx* ctx, uint32_t* support_out);

/* gc_ktruss (north star "gc_ktruss(k) returning the surviving edge mask";
 * P:247 [k-Truss] "each edge is contained in at least (k-2) triangles in the
 * same subgraph"; Alg. 4).  Computes the maximal k-truss (reading
 * A2) by batch peeling: each round removes every live edge whose support is
 * below k-2 (Alg. 4's vector x) and decrements the support of the live
 * edges of every triangle it destroys, once per triangle (reading A5), until
 * a fixed point.  Cold: includes the support computation.
 * alive_out: m uint8 (1 = edge in the k-truss), canonical order;
 * *m_alive (may be NULL) = number of surviving edges.
 * k < 2 -> GC_ERR_INVALID; k = 2 -> every edge (vacuous). */
int gc_ktruss(gc_ctx* ctx, int32_t k, uint8_t* alive_out, int64_t* m_alive);

/* gc_ktruss_analysis: the three results above from ONE support pass — the
 * north star's own chain ("for each edge (u,v), count |N(u) ∩ N(v)|.
 * Triangle counting sums this support. k-truss repeats it while peeling").
 * The support pass finds every triangle once (its hit total is the triangle
 * count, = Σ support / 3), its per-edge supports are written out, and the
 * same supports seed the k-truss peel.  Each output pointer may be NULL (not
 * written); otherwise the same layouts as gc_triangle_count (*triangles),
 * gc_edge_support (support_out, m uint32) and gc_ktruss (alive_out, m uint8;
 * *m_alive).  Cold like gc_ktruss.  k < 2 -> GC_ERR_INVALID. */
int gc_ktruss_analysis(gc_ctx* ctx, int32_t k, uint64_t* triangles, uint32_t* support_out, uint8_t* alive_out,
                       int64_t* m_alive);

/* gc_ktruss_analysis_async: gc_ktruss_analysis whose per-edge outputs
 * (support_out, alive_out) are copied back on a library copy stream: the
 * call returns once they are computed, with *triangles and *m_alive already
 * valid, while the copies run (overlapping e.g. the next gc_stage_edges /
 * gc_build_csr).  The two buffers may be read only after gc_wait returns
 * (or after the next call on this context that produces per-edge outputs,
 * which waits for them on the device before reusing its staging memory).
 * Page-locked host buffers give the overlap; pageable ones are copied
 * before return.  Arguments and errors as gc_ktruss_analysis. */
int gc_ktruss_analysis_async(gc_ctx* ctx, int32_t k, uint64_t* triangles, uint32_t* support_out,
                             uint8_t* alive_out, int64_t* m_alive);

/* gc_wait: block until every asynchronous copy of this context
 * (gc_ktruss_analysis_async outputs, a pending gc_stage_edges) is done. */
int gc_wait(gc_ctx* ctx);

/* gc_list_triangles (Alg. 1's triangle records; SURVEY §8(f)
 * NEXT #3): every triangle once as three ORIGINAL vertex ids, ascending
 * within the triple; triples in unspecified order.  tri_out: 3 * capacity
 * int32 (host or device); *count = the number of triangles T.  capacity < T
 * -> GC_ERR_RANGE with *count set and nothing written (call again with a
 * buffer of 3 * T).  Includes a triangle-count pass; runs on this rank alone
 * (every rank of a communicator lists the whole graph). */
int gc_list_triangles(gc_ctx* ctx, int32_t* tri_out, int64_t capacity, int64_t* count);

/* gc_truss_decomposition (k = 3 on the full graph, then
 * k + 1 on the result, until empty).  trussness_out[i] = largest k such that
 * canonical edge i is in the k-truss (>= 2); m int32 entries.  *kmax =
 * largest trussness, 0 when m == 0 (reading A7). */
int gc_truss_decomposition(gc_ctx* ctx, int32_t* trussness_out, int32_t* kmax);

/* ---------------------------------------------------- measurement aids --
 * Options (testing and tuning; defaults are the production settings). */
typedef enum gc_option {
    GC_OPT_FORCE_CLASS = 1,   /* -1 auto; 0..3 force every oriented edge through one
                                 intersection kernel class */
    GC_OPT_TASK_CHUNK = 2,    /* cost budget per intersection task, in units of one wedge
                                 plus 128 per in-edge (default 32768; 8x for block tasks) */
    GC_OPT_TIMING = 3,        /* 1: record CUDA events per phase (default 1) */
    GC_OPT_LONG_SEG = 5,      /* suffixes at least this long take the warp-vector path
                                 (default 48; 2^30 disables it; testing) */
    GC_OPT_BLOCK_BATCH = 6,   /* heavy-head kernel: consecutive tasks per block batch,
                                 batches dealt round-robin (default 32; tuning) */
    GC_OPT_BLOCK_BITMAP = 4,  /* 1: heavy-head kernel may use the rank-window bitmap
                                 (default); 0: always its hash table (testing) */
    GC_OPT_SUP_SKIP = 7,      /* timing diagnostics only (wrong supports when nonzero):
                                 mask of support roles to skip, 1 (u,w), 2 (v,w),
                                 4 (u,v); default 0.  A nonzero value is refused with
                                 GC_ERR_INVALID unless the environment has GC_DIAG=1 */
    GC_OPT_PEEL_PART = 8,     /* 1: use the partitioned k-truss peeler (removed-edge
                                 bitmap per round, owner-only decrements; the multi-GPU
                                 path) even on a single rank (testing); it is always
                                 used when nranks > 1 or under loopback partitions */
    GC_OPT_HUGE_MAX = 9,      /* class-3 heads with d+ above this (default 8192, the
                                 16384-slot shared hash at load 1/2) search N+(v) in
                                 global memory instead (0..8192; testing) */
    GC_OPT_COMPACT = 10,      /* peeler: drop dead entries from the adjacency rows each
                                 time the live edge count falls to (value-1)/value of the
                                 last compaction during gc_truss_decomposition (default 5,
                                 i.e. 4/5; a single k-truss uses min(value, 2)); 0 or 1: never.
                                 (Before round 2 a value v meant "at 1/v"; 2 means the same
                                 in both readings, 3 now means 2/3 instead of 1/3.) */
    GC_OPT_OVERLAP = 13,      /* 1: the warp-task intersection kernels run on a library
                                 side stream that overlaps the block-task kernels and is
                                 joined before the call returns (default); 0: one stream */
    GC_OPT_GROUP_PEEL = 12,   /* peeler: rounds with at least this many frontier edges
                                 (default 0: never; 2^20 was the earlier default, slower since
                                 the per-edge search keeps two searches in flight) group
                                 their heavy edges by the endpoint with the longer live row,
                                 whose row is staged once per group as a shared-memory bitmap */
    GC_OPT_GROUP_HEAVY = 14,  /* ... heavy = shorter live row at least this long (default
                                 1024); lighter edges keep the per-edge search */
    GC_OPT_WORK_STATS = 15,   /* 1: the single-rank peeler also counts the k-truss byte
                                 model's terms (gc_stats peel_sum_min,
                                 peel_decrements) at the cost of a few small kernels per
                                 round (default 0; measurement) */
    GC_OPT_SORT_FRONT = 18,   /* peeler: a round whose frontier has at least this many edges
                                 (known on the host) is first sorted by the endpoint whose live
                                 row the per-edge search probes (default 2^20; 0: never;
                                 C4 k = 4 / 6 peel -4 % / -5 %, decomposition -2 %) */
    GC_OPT_BUILD_PART = 16,   /* gc_build_csr across owners: -1 (default)
                                 partitioned when there are several owners (NCCL ranks or
                                 loopback parts), 1 always (one owner included; testing),
                                 0 never (every rank builds the whole CSR) */
} gc_option;
int gc_set_option(gc_ctx* ctx, int option, int64_t value);

/* Statistics of the most recent calls (device times from CUDA events on the
 * context stream, milliseconds). */
typedef struct gc_stats {
    double build_ms;          /* last gc_build_csr */
    double tc_ms;             /* last gc_triangle_count (excluding output copy) */
    double tc_kernel_ms;      /* intersection kernels of that call */
    double support_ms;        /* last gc_edge_support */
    double support_kernel_ms; /* support intersection kernels of that call */
    double ktruss_ms;         /* last gc_ktruss (support + peel) */
    double peel_ms;           /* peel part of the last gc_ktruss / decomposition */
    double decomp_ms;         /* last gc_truss_decomposition */
    double peel_kernel_ms;    /* triangle-destroying kernels of the last peel (sum) */
    double scan_ms;           /* level frontier scans of the last peel (sum) */
    double compact_ms;        /* dead-entry compactions of the last peel (sum) */
    int64_t launches;         /* libgc kernel launches since gc_reset_stats */
    int64_t lib_launches;     /* CUB (library) kernel launches, estimated, same window */
    int64_t peel_rounds;      /* rounds of the last peel (ktruss or decomposition) */
    int64_t compactions;      /* dead-entry compactions of the last peel */
    int64_t n, m;
    int64_t wedges;           /* sum over vertices of C(d+(x), 2): intersection work */
    int64_t q_out;            /* sum d+(x)^2   (SURVEY §8(d) byte model) */
    int64_t q_in;             /* sum d-(x) d+(x) */
    int64_t max_out_degree;   /* max d+ */
    int64_t max_degree;       /* max d */
    int64_t tasks[5];         /* intersection tasks per kernel class (last build): 0 lane, 1 warp,
                                 2 block (bitmap or hash), 3 huge (hash), 4 wide bitmap */
    int64_t aux[8];           /* heads with d+ > 256 by rank span of N+ (<=2^17, 2^18,
                                 2^19, more): counts [0..3], in-degree weighted [4..7] */
    int64_t peel_sum_min;     /* GC_OPT_WORK_STATS, last peel: sum over rounds, over frontier
                                 edges (a,b) with support > 0, of min(d(a), d(b)) (alive
                                 degrees at the round start); -1 when not counted */
    int64_t peel_decrements;  /* ... support decrements D applied to surviving edges; -1 */
    double part_ms[16];       /* loopback partitions: intersection-kernel time of each virtual
                                 rank in the last triangle-count / support pass (balance of
                                 the 1D cost cut; ranks >= 16 not recorded) */
    double part_build_ms[16]; /* loopback partitions: device time of each virtual rank's share
                                 of the last partitioned gc_build_csr (its three sorts) */
} gc_stats;
int gc_get_stats(const gc_ctx* ctx, gc_stats* out);
int gc_reset_stats(gc_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GC_H_ */
