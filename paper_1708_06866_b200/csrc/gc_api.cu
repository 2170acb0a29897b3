// gc_api.cu — the extern "C" entry points of include/gc.h and the context
// plumbing (errors, stream-ordered buffers, host<->device copies).
#include <cstring>
#include <new>

#include <utility>

#include "gc_internal.cuh"
#include <nvtx3/nvToolsExt.h>

// NVTX range around every compute entry point (header-only NVTX v3: a no-op
// unless a profiler injects itself; ncu --nvtx / nsys show the API calls)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

namespace gcx {

int fail(gc_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

int cuda_fail(gc_ctx* c, cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    snprintf(buf, sizeof(buf), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
             cudaGetErrorString(e), what, file, line);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();  // clear the sticky-free allocation error
        return fail(c, GC_ERR_OOM, buf);
    }
    if (c) c->poisoned = true;
    return fail(c, GC_ERR_CUDA, buf);
}

int ensure(gc_ctx* c, Buf& b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return GC_OK;
    if (b.p) {
        GC_CUDA(c, cudaFreeAsync(b.p, c->stream));
        b.p = nullptr;
        b.cap = 0;
    }
    size_t want = bytes + bytes / 8;  // slack so growing configs do not thrash
    cudaError_t e = c->pool ? cudaMallocFromPoolAsync(&b.p, want, c->pool, c->stream)
                            : cudaMallocAsync(&b.p, want, c->stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        // retry without slack
        e = c->pool ? cudaMallocFromPoolAsync(&b.p, bytes, c->pool, c->stream)
                    : cudaMallocAsync(&b.p, bytes, c->stream);
        if (e != cudaSuccess) {
            cudaGetLastError();
            b.p = nullptr;
            char msg[128];
            snprintf(msg, sizeof(msg), "device allocation of %zu bytes failed", bytes);
            return fail(c, GC_ERR_OOM, msg);
        }
        want = bytes;
    }
    b.cap = want;
    return GC_OK;
}

void release(gc_ctx* c, Buf& b) {
    if (b.p) cudaFreeAsync(b.p, c->stream);
    b.p = nullptr;
    b.cap = 0;
}

int host_scratch(gc_ctx* c, size_t bytes) {
    if (c->hpin_cap >= bytes) return GC_OK;
    if (c->hpin) cudaFreeHost(c->hpin);
    c->hpin = nullptr;
    c->hpin_cap = 0;
    GC_CUDA(c, cudaHostAlloc(&c->hpin, bytes, cudaHostAllocMapped));
    GC_CUDA(c, cudaHostGetDevicePointer(&c->hpin_dev, c->hpin, 0));
    c->hpin_cap = bytes;
    return GC_OK;
}

int sync(gc_ctx* c) {
    GC_CUDA(c, cudaStreamSynchronize(c->stream));
    return GC_OK;
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int copy_out(gc_ctx* c, void* dst, const void* src_dev, size_t nbytes) {
    if (nbytes == 0) return GC_OK;
    cudaMemcpyKind kind = is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    GC_CUDA(c, cudaMemcpyAsync(dst, src_dev, nbytes, kind, c->stream));
    return GC_OK;
}

__global__ void k_read_small(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

int read_small(gc_ctx* c, void* host_dst, const void* src_dev, size_t nbytes) {
    // host_dst lies in the context's page-locked scratch, mapped into the
    // device address space: one tiny kernel writes it, so the read needs no
    // copy engine (whose FIFO may hold a long asynchronous read-back)
    char* h = static_cast<char*>(host_dst);
    char* base = static_cast<char*>(c->hpin);
    if (!c->hpin_dev || h < base || h + nbytes > base + c->hpin_cap || nbytes > 4096) {
        GC_CUDA(c, cudaMemcpyAsync(host_dst, src_dev, nbytes, cudaMemcpyDeviceToHost, c->stream));
        return GC_OK;
    }
    k_read_small<<<1, 128, 0, c->stream>>>(static_cast<const uint8_t*>(src_dev),
                                           reinterpret_cast<uint8_t*>(static_cast<char*>(c->hpin_dev) + (h - base)),
                                           (int)nbytes);
    GC_CUDA(c, cudaGetLastError());
    ++c->stats.launches;
    return GC_OK;
}

int copy_out_staged(gc_ctx* c, void* dst, const void* src_dev, size_t nbytes) {
    if (!c->async_out) return copy_out(c, dst, src_dev, nbytes);
    if (nbytes == 0) return GC_OK;
    if (!c->d2h_s) {
        GC_CUDA(c, cudaStreamCreateWithFlags(&c->d2h_s, cudaStreamNonBlocking));
        GC_CUDA(c, cudaEventCreateWithFlags(&c->ev_out_ready, cudaEventDisableTiming));
        GC_CUDA(c, cudaEventCreateWithFlags(&c->ev_d2h_done, cudaEventDisableTiming));
    }
    GC_CUDA(c, cudaEventRecord(c->ev_out_ready, c->stream));
    GC_CUDA(c, cudaStreamWaitEvent(c->d2h_s, c->ev_out_ready, 0));
    // a copy engine: the context stream's own small reads (read_small) do
    // not queue behind it, and the SMs stay free for the next call's kernels
    GC_CUDA(c, cudaMemcpyAsync(dst, src_dev, nbytes, cudaMemcpyDefault, c->d2h_s));
    GC_CUDA(c, cudaEventRecord(c->ev_d2h_done, c->d2h_s));
    c->d2h_pending = true;
    return GC_OK;
}

int claim_out(gc_ctx* c) {
    if (c->d2h_pending) GC_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_d2h_done, 0));
    return GC_OK;
}

int copy_in(gc_ctx* c, void* dst_dev, const void* src, size_t nbytes) {
    if (nbytes == 0) return GC_OK;
    cudaMemcpyKind kind = is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    GC_CUDA(c, cudaMemcpyAsync(dst_dev, src, nbytes, kind, c->stream));
    return GC_OK;
}

int record(gc_ctx* c, int i) {
    if (!c->timing) return GC_OK;
    GC_CUDA(c, cudaEventRecord(c->ev[i], c->stream));
    return GC_OK;
}

float elapsed(gc_ctx* c, int a, int b) {
    if (!c->timing) return 0.f;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]) != cudaSuccess) {
        cudaGetLastError();
        return 0.f;
    }
    return ms;
}

}  // namespace gcx

using namespace gcx;

static int check_ctx(const gc_ctx* c) {
    if (!c) return GC_ERR_INVALID;
    if (c->poisoned) return GC_ERR_STATE;
    return GC_OK;
}

static thread_local std::string g_create_err;

static bool diag_enabled() {
    const char* e = getenv("GC_DIAG");
    return e && e[0] == '1';
}

extern "C" {

int gc_create(gc_ctx** out, int device, void* cuda_stream) {
    if (!out) return GC_ERR_INVALID;
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        g_create_err = std::string("gc_create: no CUDA device ") + std::to_string(device) +
                       (e != cudaSuccess ? std::string(" (") + cudaGetErrorString(e) + ")" : "");
        return e != cudaSuccess ? GC_ERR_CUDA : GC_ERR_INVALID;
    }
    gc_ctx* c = new (std::nothrow) gc_ctx();
    if (!c) return GC_ERR_OOM;
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        g_create_err = "gc_create: cudaSetDevice failed";
        delete c;
        return GC_ERR_CUDA;
    }
    if (cuda_stream) {
        c->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
            g_create_err = "gc_create: cudaStreamCreate failed";
            delete c;
            return GC_ERR_CUDA;
        }
        c->own_stream = true;
    }
    // a library-owned pool that keeps freed memory cached (steady-state steps
    // then allocate nothing); the device's default pool is left untouched and
    // everything this pool holds is returned by gc_destroy
    {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        if (cudaMemPoolCreate(&c->pool, &props) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr);
        } else {
            c->pool = nullptr;      // fall back to the default pool's stream-ordered allocator
        }
    }
    for (auto& ev : c->ev) cudaEventCreate(&ev);
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)
        c->side = nullptr;          // no overlap: everything stays on the context stream
    cudaGetLastError();
    *out = c;
    return GC_OK;
}

int gc_destroy(gc_ctx* c) {
    if (!c) return GC_OK;
    cudaSetDevice(c->device);
    if (c->copy_s) cudaStreamSynchronize(c->copy_s);
    if (c->d2h_s) cudaStreamSynchronize(c->d2h_s);
    cudaStreamSynchronize(c->stream);
    gcx::Buf* bufs[] = {&c->raw_u, &c->raw_v, &c->stage_u, &c->stage_v, &c->canon, &c->deg, &c->rank_of, &c->dag_ptr,
                        &c->dag_col, &c->dag_src, &c->dag_eid, &c->in_ptr, &c->in_pos, &c->in_src,
                        &c->in_dst, &c->task_i0, &c->task_i1, &c->in_cost, &c->tmp_a, &c->tmp_b, &c->keys_a, &c->keys_b,
                        &c->vals_a, &c->vals_b, &c->cub_tmp, &c->scal, &c->sup, &c->uw16, &c->out_tmp, &c->out_tmp2, &c->id_of, &c->list_out, &c->batch_slot, &c->grp_keys, &c->grp_vals, &c->grp_starts, &c->grp_flags, &c->grp_light,
                        &c->sym_ptr, &c->sym_col, &c->sym_eid, &c->alive, &c->front_a,
                        &c->front_b, &c->tau, &c->xbits, &c->nbits, &c->zbits, &c->sup_parts, &c->live_len, &c->long_rows, &c->alist,
                        &c->vdeg, &c->zlist, &c->task_pref, &c->dec_out, &c->dec_in};
    for (auto* b : bufs) release(c, *b);
    cudaStreamSynchronize(c->stream);
    if (c->pool) cudaMemPoolDestroy(c->pool);   // returns the cached blocks to the device
    nccl_destroy(c);
    if (c->hpin) cudaFreeHost(c->hpin);
    for (auto& ev : c->ev)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : c->pev)
        if (ev) cudaEventDestroy(ev);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->copy_s) cudaStreamDestroy(c->copy_s);
    if (c->d2h_s) cudaStreamDestroy(c->d2h_s);
    if (c->ev_out_ready) cudaEventDestroy(c->ev_out_ready);
    if (c->ev_d2h_done) cudaEventDestroy(c->ev_d2h_done);
    if (c->ev_staged) cudaEventDestroy(c->ev_staged);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    cudaGetLastError();
    delete c;
    return GC_OK;
}

const char* gc_last_error(const gc_ctx* c) {
    if (!c) return g_create_err.c_str();
    return c->err.c_str();
}

int gc_nccl_unique_id(void* id_out) {
    if (!id_out) return GC_ERR_INVALID;
    return nccl_get_unique_id(id_out);
}

int gc_comm_init(gc_ctx* c, const void* id, int nranks, int rank) {
    GC_TRY(check_ctx(c));
    if (!id || nranks < 1 || rank < 0 || rank >= nranks) return fail(c, GC_ERR_INVALID, "gc_comm_init: bad arguments");
    if (c->state != 0) return fail(c, GC_ERR_STATE, "gc_comm_init must precede gc_load_edges");
    if (c->nccl || c->loop_parts) return fail(c, GC_ERR_STATE, "communicator already initialised");
    cudaSetDevice(c->device);
    // nranks == 1 forms a real one-rank communicator: every collective of the
    // multi-GPU path (allreduce, in-place allgather) then runs through NCCL
    return nccl_init(c, id, nranks, rank);
}

int gc_partition_bounds(const int64_t* pref, int64_t len, int nparts, int64_t* bounds) {
    if (!pref || !bounds || len < 0 || nparts < 1) return GC_ERR_INVALID;
    const int64_t total = pref[len];
    // owner(i) = floor(pref[i] * nparts / total) is nondecreasing in i
    int64_t i = 0;
    for (int r = 0; r < nparts; ++r) {
        if (total <= 0) {
            bounds[r] = r == 0 ? 0 : len;
            continue;
        }
        while (i < len && (pref[i] * (int64_t)nparts) / total < r) ++i;
        bounds[r] = i;
    }
    bounds[nparts] = len;
    return GC_OK;
}

int gc_comm_init_loopback(gc_ctx* c, int nparts) {
    GC_TRY(check_ctx(c));
    if (nparts < 1 || nparts > 64) return fail(c, GC_ERR_INVALID, "gc_comm_init_loopback: nparts must be 1..64");
    if (c->state != 0) return fail(c, GC_ERR_STATE, "gc_comm_init_loopback must precede gc_load_edges");
    if (c->nccl) return fail(c, GC_ERR_STATE, "communicator already initialised");
    c->loop_parts = nparts;
    c->nranks = 1;
    c->rank = 0;
    return GC_OK;
}

// wait for a pending gc_stage_edges copy (it may still read the caller's buffers)
static int drain_stage(gc_ctx* c) {
    if (c->copy_s) GC_CUDA(c, cudaStreamSynchronize(c->copy_s));
    return GC_OK;
}

int gc_stage_edges(gc_ctx* c, const int32_t* u, const int32_t* v, int64_t nnz) {
    NvtxRange nvtx_range("gc_stage_edges");
    GC_TRY(check_ctx(c));
    if (nnz < 0 || (nnz > 0 && (!u || !v))) return fail(c, GC_ERR_INVALID, "gc_stage_edges: bad arguments");
    cudaSetDevice(c->device);
    if (!c->copy_s) {
        GC_CUDA(c, cudaStreamCreateWithFlags(&c->copy_s, cudaStreamNonBlocking));
        GC_CUDA(c, cudaEventCreateWithFlags(&c->ev_staged, cudaEventDisableTiming));
    }
    GC_TRY(drain_stage(c));
    c->stage_nnz = -1;
    GC_TRY(ensure(c, c->stage_u, (size_t)nnz * sizeof(int32_t)));   // allocation is ordered on the context stream
    GC_TRY(ensure(c, c->stage_v, (size_t)nnz * sizeof(int32_t)));
    GC_CUDA(c, cudaEventRecord(c->ev_staged, c->stream));            // buffers ready before the copy
    GC_CUDA(c, cudaStreamWaitEvent(c->copy_s, c->ev_staged, 0));
    if (nnz > 0) {
        GC_CUDA(c, cudaMemcpyAsync(c->stage_u.p, u, (size_t)nnz * 4, cudaMemcpyDefault, c->copy_s));
        GC_CUDA(c, cudaMemcpyAsync(c->stage_v.p, v, (size_t)nnz * 4, cudaMemcpyDefault, c->copy_s));
    }
    GC_CUDA(c, cudaEventRecord(c->ev_staged, c->copy_s));
    c->stage_nnz = nnz;
    if (c->state < 1) c->state = 1;   // gc_build_csr may follow directly
    return GC_OK;
}

int gc_load_edges(gc_ctx* c, const int32_t* u, const int32_t* v, int64_t nnz) {
    NvtxRange nvtx_range("gc_load_edges");
    GC_TRY(check_ctx(c));
    if (nnz < 0 || (nnz > 0 && (!u || !v))) return fail(c, GC_ERR_INVALID, "gc_load_edges: bad arguments");
    cudaSetDevice(c->device);
    GC_TRY(drain_stage(c));
    c->stage_nnz = -1;
    GC_TRY(ensure(c, c->raw_u, (size_t)nnz * sizeof(int32_t)));
    GC_TRY(ensure(c, c->raw_v, (size_t)nnz * sizeof(int32_t)));
    GC_TRY(copy_in(c, c->raw_u.p, u, (size_t)nnz * sizeof(int32_t)));
    GC_TRY(copy_in(c, c->raw_v.p, v, (size_t)nnz * sizeof(int32_t)));
    GC_TRY(sync(c));
    c->nnz = nnz;
    c->state = 1;
    c->tasks_ready = false;
    c->sym_ready = false;
    c->n = c->m = 0;
    return GC_OK;
}

int gc_build_csr(gc_ctx* c) {
    NvtxRange nvtx_range("gc_build_csr");
    GC_TRY(check_ctx(c));
    if (c->state < 1) return fail(c, GC_ERR_STATE, "gc_build_csr before gc_load_edges");
    cudaSetDevice(c->device);
    if (c->stage_nnz >= 0) {
        // a staged list: the context stream waits for its copy, then the
        // staged and current raw buffers trade places
        GC_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_staged, 0));
        std::swap(c->raw_u, c->stage_u);
        std::swap(c->raw_v, c->stage_v);
        c->nnz = c->stage_nnz;
        c->stage_nnz = -1;
    }
    c->state = 1;
    c->tasks_ready = false;
    c->sym_ready = false;
    c->n = c->m = 0;
    GC_TRY(record(c, 0));
    GC_TRY(build_csr(c));
    GC_TRY(prepare_tasks(c));
    GC_TRY(record(c, 1));
    GC_TRY(sync(c));
    c->stats.build_ms = elapsed(c, 0, 1);
    c->state = 2;
    return GC_OK;
}

int gc_num_vertices(const gc_ctx* c, int64_t* n) {
    GC_TRY(check_ctx(c));
    if (!n) return GC_ERR_INVALID;
    if (c->state < 2) return GC_ERR_STATE;
    *n = c->n;
    return GC_OK;
}

int gc_num_edges(const gc_ctx* c, int64_t* m) {
    GC_TRY(check_ctx(c));
    if (!m) return GC_ERR_INVALID;
    if (c->state < 2) return GC_ERR_STATE;
    *m = c->m;
    return GC_OK;
}

int gc_triangle_count(gc_ctx* c, uint64_t* count) {
    NvtxRange nvtx_range("gc_triangle_count");
    GC_TRY(check_ctx(c));
    if (!count) return fail(c, GC_ERR_INVALID, "gc_triangle_count: NULL output");
    if (c->state < 2) return fail(c, GC_ERR_STATE, "gc_triangle_count before gc_build_csr");
    cudaSetDevice(c->device);
    return triangle_count(c, count);
}

int gc_edge_support(gc_ctx* c, uint32_t* support_out) {
    NvtxRange nvtx_range("gc_edge_support");
    GC_TRY(check_ctx(c));
    if (c->state < 2) return fail(c, GC_ERR_STATE, "gc_edge_support before gc_build_csr");
    if (!support_out && c->m > 0) return fail(c, GC_ERR_INVALID, "gc_edge_support: NULL output");
    cudaSetDevice(c->device);
    GC_TRY(claim_out(c));   // a pending asynchronous read-back still reads out_tmp / out_tmp2
    GC_TRY(record(c, 4));
    GC_TRY(support_dag(c));
    GC_TRY(ensure(c, c->out_tmp, (size_t)c->m * sizeof(uint32_t)));
    GC_TRY(scatter_canonical_u32(c, c->sup.as<uint32_t>(), c->out_tmp.as<uint32_t>()));
    GC_TRY(record(c, 5));
    GC_TRY(copy_out(c, support_out, c->out_tmp.p, (size_t)c->m * sizeof(uint32_t)));
    GC_TRY(sync(c));
    c->stats.support_ms = elapsed(c, 4, 5);
    c->stats.support_kernel_ms = elapsed(c, 6, 7);
    return GC_OK;
}

int gc_ktruss(gc_ctx* c, int32_t k, uint8_t* alive_out, int64_t* m_alive) {
    NvtxRange nvtx_range("gc_ktruss");
    GC_TRY(check_ctx(c));
    if (k < 2) return fail(c, GC_ERR_INVALID, "gc_ktruss: k must be >= 2 (P:280)");
    if (c->state < 2) return fail(c, GC_ERR_STATE, "gc_ktruss before gc_build_csr");
    if (!alive_out && c->m > 0) return fail(c, GC_ERR_INVALID, "gc_ktruss: NULL output");
    cudaSetDevice(c->device);
    GC_TRY(claim_out(c));   // a pending asynchronous read-back still reads out_tmp / out_tmp2
    return ktruss(c, k, alive_out, m_alive);
}

int gc_ktruss_analysis(gc_ctx* c, int32_t k, uint64_t* triangles, uint32_t* support_out, uint8_t* alive_out,
                       int64_t* m_alive) {
    NvtxRange nvtx_range("gc_ktruss_analysis");
    GC_TRY(check_ctx(c));
    if (k < 2) return fail(c, GC_ERR_INVALID, "gc_ktruss_analysis: k must be >= 2 (P:280)");
    if (c->state < 2) return fail(c, GC_ERR_STATE, "gc_ktruss_analysis before gc_build_csr");
    cudaSetDevice(c->device);
    GC_TRY(claim_out(c));   // a pending asynchronous read-back still reads out_tmp / out_tmp2
    return ktruss_analysis(c, k, triangles, support_out, alive_out, m_alive);
}

int gc_ktruss_analysis_async(gc_ctx* c, int32_t k, uint64_t* triangles, uint32_t* support_out, uint8_t* alive_out,
                             int64_t* m_alive) {
    NvtxRange nvtx_range("gc_ktruss_analysis_async");
    GC_TRY(check_ctx(c));
    if (k < 2) return fail(c, GC_ERR_INVALID, "gc_ktruss_analysis_async: k must be >= 2 (P:280)");
    if (c->state < 2) return fail(c, GC_ERR_STATE, "gc_ktruss_analysis_async before gc_build_csr");
    cudaSetDevice(c->device);
    GC_TRY(claim_out(c));   // a pending asynchronous read-back still reads out_tmp / out_tmp2
    c->async_out = true;
    const int rc = ktruss_analysis(c, k, triangles, support_out, alive_out, m_alive);
    c->async_out = false;
    return rc;
}

int gc_wait(gc_ctx* c) {
    GC_TRY(check_ctx(c));
    cudaSetDevice(c->device);
    if (c->d2h_s) GC_CUDA(c, cudaStreamSynchronize(c->d2h_s));
    if (c->copy_s) GC_CUDA(c, cudaStreamSynchronize(c->copy_s));
    c->d2h_pending = false;
    return GC_OK;
}

int gc_truss_decomposition(gc_ctx* c, int32_t* tau_out, int32_t* kmax) {
    NvtxRange nvtx_range("gc_truss_decomposition");
    GC_TRY(check_ctx(c));
    if (c->state < 2) return fail(c, GC_ERR_STATE, "gc_truss_decomposition before gc_build_csr");
    if (!kmax || (!tau_out && c->m > 0)) return fail(c, GC_ERR_INVALID, "gc_truss_decomposition: NULL output");
    cudaSetDevice(c->device);
    GC_TRY(claim_out(c));   // a pending asynchronous read-back still reads out_tmp / out_tmp2
    return truss_decomposition(c, tau_out, kmax);
}

int gc_set_option(gc_ctx* c, int option, int64_t value) {
    GC_TRY(check_ctx(c));
    switch (option) {
        case GC_OPT_FORCE_CLASS:
            if (value < -1 || value > 3) return fail(c, GC_ERR_INVALID, "force class must be -1..3");
            c->force_class = (int)value;
            c->tasks_ready = false;
            if (c->state == 2) {
                cudaSetDevice(c->device);
                GC_TRY(prepare_tasks(c));
                GC_TRY(sync(c));
            }
            return GC_OK;
        case GC_OPT_TASK_CHUNK:
            if (value < 32 || value > (int64_t)1 << 30) return fail(c, GC_ERR_INVALID, "task chunk out of range");
            c->task_chunk = value;
            c->tasks_ready = false;
            if (c->state == 2) {
                cudaSetDevice(c->device);
                GC_TRY(prepare_tasks(c));
                GC_TRY(sync(c));
            }
            return GC_OK;
        case GC_OPT_BLOCK_BATCH:
            if (value < 1 || value > (1 << 20)) return fail(c, GC_ERR_INVALID, "block batch must be 1..2^20");
            c->block_batch = (int)value;
            return GC_OK;
        case GC_OPT_LONG_SEG:
            if (value < 1) return fail(c, GC_ERR_INVALID, "long segment threshold must be >= 1");
            c->long_seg = value > (1 << 30) ? (1 << 30) : (int)value;
            return GC_OK;
        case GC_OPT_BLOCK_BITMAP:
            c->block_bitmap = value ? 1 : 0;
            c->tasks_ready = false;   // the class of a head depends on the bitmap capacity
            if (c->state == 2) {
                cudaSetDevice(c->device);
                GC_TRY(prepare_tasks(c));
                GC_TRY(sync(c));
            }
            return GC_OK;
        case GC_OPT_SUP_SKIP:
            // diagnostics only: skipped roles give wrong supports, so the option
            // is refused unless the process opted in with GC_DIAG=1
            if (value != 0 && !diag_enabled())
                return fail(c, GC_ERR_INVALID, "GC_OPT_SUP_SKIP is a timing diagnostic (wrong supports); set GC_DIAG=1 to allow it");
            if (value < 0 || value > 7) return fail(c, GC_ERR_INVALID, "support skip mask must be 0..7");
            c->sup_skip = (int)value;
            return GC_OK;
        case GC_OPT_HUGE_MAX:
            if (value < 0 || value > 8192) return fail(c, GC_ERR_INVALID, "huge-head hash limit must be 0..8192");
            c->huge_max = (int)value;
            return GC_OK;
        case GC_OPT_COMPACT:
            if (value < 0 || value > 1024) return fail(c, GC_ERR_INVALID, "compaction divisor must be 0..1024");
            c->compact_div = (int)value;
            return GC_OK;
        case GC_OPT_OVERLAP:
            c->overlap = value ? 1 : 0;
            return GC_OK;
        case GC_OPT_GROUP_PEEL:
            if (value < 0 || value > ((int64_t)1 << 30)) return fail(c, GC_ERR_INVALID, "group threshold out of range");
            c->group_peel = (int)value;
            return GC_OK;
        case GC_OPT_GROUP_HEAVY:
            if (value < 1 || value > ((int64_t)1 << 30)) return fail(c, GC_ERR_INVALID, "heavy row bound out of range");
            c->group_heavy = (int)value;
            return GC_OK;
        case GC_OPT_PEEL_PART:
            c->peel_part = value ? 1 : 0;
            return GC_OK;
        case GC_OPT_BUILD_PART:
            if (value < -1 || value > 1) return fail(c, GC_ERR_INVALID, "build partition mode must be -1, 0 or 1");
            c->build_part = (int)value;
            return GC_OK;
        case GC_OPT_SORT_FRONT:
            if (value < 0 || value > ((int64_t)1 << 30)) return fail(c, GC_ERR_INVALID, "sort threshold out of range");
            c->sort_front = (int)value;
            return GC_OK;
        case GC_OPT_WORK_STATS:
            c->work_stats = value ? 1 : 0;
            return GC_OK;
        case GC_OPT_TIMING:
            c->timing = value ? 1 : 0;
            return GC_OK;
        default:
            return fail(c, GC_ERR_INVALID, "unknown option");
    }
}

int gc_get_stats(const gc_ctx* c, gc_stats* out) {
    if (!c || !out) return GC_ERR_INVALID;
    *out = c->stats;
    return GC_OK;
}

int gc_reset_stats(gc_ctx* c) {
    if (!c) return GC_ERR_INVALID;
    c->stats.launches = 0;
    c->stats.lib_launches = 0;
    return GC_OK;
}

}  // extern "C"
