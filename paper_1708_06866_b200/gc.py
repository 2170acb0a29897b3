"""Thin ctypes binding of libgc (include/gc.h) — argument marshalling only.

Every step of the path runs in libgc's CUDA kernels; this module converts
numpy arrays / torch tensors to pointers and status codes to exceptions.
There is no CPU fallback: if ``libgc.so`` is missing or no GPU is present the
calls raise.

The module exports the C entry points under their C names (``gc_create``,
``gc_load_edges``, ..., bound with argtypes) plus ``Context``, a small object
wrapper used by the tests and bench.py.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GC_LIB_PATH") or os.path.join(_HERE, "libgc.so")   # override: tuning builds

GC_OK = 0
GC_ERR_INVALID = 1
GC_ERR_STATE = 2
GC_ERR_RANGE = 3
GC_ERR_OOM = 4
GC_ERR_CUDA = 5
GC_ERR_NCCL = 6
_NAMES = {0: "GC_OK", 1: "GC_ERR_INVALID", 2: "GC_ERR_STATE", 3: "GC_ERR_RANGE", 4: "GC_ERR_OOM",
          5: "GC_ERR_CUDA", 6: "GC_ERR_NCCL"}

GC_OPT_FORCE_CLASS = 1
GC_OPT_TASK_CHUNK = 2
GC_OPT_TIMING = 3
GC_OPT_BLOCK_BITMAP = 4
GC_OPT_LONG_SEG = 5
GC_OPT_BLOCK_BATCH = 6
GC_OPT_SUP_SKIP = 7
GC_OPT_PEEL_PART = 8
GC_OPT_HUGE_MAX = 9
GC_OPT_COMPACT = 10
GC_OPT_GROUP_PEEL = 12
GC_OPT_GROUP_HEAVY = 14
GC_OPT_OVERLAP = 13
GC_OPT_WORK_STATS = 15
GC_OPT_BUILD_PART = 16
GC_OPT_SORT_FRONT = 18

# Every symbol include/gc.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "gc_create", "gc_destroy", "gc_last_error", "gc_nccl_unique_id", "gc_comm_init",
    "gc_comm_init_loopback", "gc_load_edges", "gc_stage_edges", "gc_build_csr", "gc_ktruss_analysis_async", "gc_wait", "gc_num_vertices", "gc_num_edges",
    "gc_get_edges", "gc_triangle_count", "gc_edge_support", "gc_ktruss", "gc_ktruss_analysis",
    "gc_truss_decomposition", "gc_list_triangles",
    "gc_set_option", "gc_get_stats", "gc_reset_stats", "gc_partition_bounds",
]


class gc_stats(ctypes.Structure):
    _fields_ = [
        ("build_ms", ctypes.c_double), ("tc_ms", ctypes.c_double), ("tc_kernel_ms", ctypes.c_double),
        ("support_ms", ctypes.c_double), ("support_kernel_ms", ctypes.c_double),
        ("ktruss_ms", ctypes.c_double), ("peel_ms", ctypes.c_double), ("decomp_ms", ctypes.c_double),
        ("peel_kernel_ms", ctypes.c_double), ("scan_ms", ctypes.c_double), ("compact_ms", ctypes.c_double),
        ("launches", ctypes.c_int64), ("lib_launches", ctypes.c_int64), ("peel_rounds", ctypes.c_int64),
        ("compactions", ctypes.c_int64),
        ("n", ctypes.c_int64), ("m", ctypes.c_int64), ("wedges", ctypes.c_int64),
        ("q_out", ctypes.c_int64), ("q_in", ctypes.c_int64), ("max_out_degree", ctypes.c_int64),
        ("max_degree", ctypes.c_int64), ("tasks", ctypes.c_int64 * 5),
        ("aux", ctypes.c_int64 * 8),
        ("peel_sum_min", ctypes.c_int64), ("peel_decrements", ctypes.c_int64),
        ("part_ms", ctypes.c_double * 16), ("part_build_ms", ctypes.c_double * 16),
    ]


class GcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


_LIB = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libgc.so (fails loudly: there is no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(f"libgc.so not built at {path}: run `make gc` or __graft_entry__.build()")
    L = ctypes.CDLL(path)
    sig = {
        "gc_create": ([ctypes.POINTER(_vp), ctypes.c_int, _vp], ctypes.c_int),
        "gc_destroy": ([_vp], ctypes.c_int),
        "gc_last_error": ([_vp], ctypes.c_char_p),
        "gc_nccl_unique_id": ([_vp], ctypes.c_int),
        "gc_comm_init": ([_vp, _vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "gc_comm_init_loopback": ([_vp, ctypes.c_int], ctypes.c_int),
        "gc_load_edges": ([_vp, _vp, _vp, _i64], ctypes.c_int),
        "gc_stage_edges": ([_vp, _vp, _vp, _i64], ctypes.c_int),
        "gc_build_csr": ([_vp], ctypes.c_int),
        "gc_num_vertices": ([_vp, ctypes.POINTER(_i64)], ctypes.c_int),
        "gc_num_edges": ([_vp, ctypes.POINTER(_i64)], ctypes.c_int),
        "gc_get_edges": ([_vp, _vp, _vp], ctypes.c_int),
        "gc_triangle_count": ([_vp, ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
        "gc_edge_support": ([_vp, _vp], ctypes.c_int),
        "gc_ktruss": ([_vp, _i32, _vp, ctypes.POINTER(_i64)], ctypes.c_int),
        "gc_ktruss_analysis": ([_vp, _i32, ctypes.POINTER(ctypes.c_uint64), _vp, _vp, ctypes.POINTER(_i64)],
                               ctypes.c_int),
        "gc_ktruss_analysis_async": ([_vp, _i32, ctypes.POINTER(ctypes.c_uint64), _vp, _vp, ctypes.POINTER(_i64)],
                                     ctypes.c_int),
        "gc_wait": ([_vp], ctypes.c_int),
        "gc_truss_decomposition": ([_vp, _vp, ctypes.POINTER(_i32)], ctypes.c_int),
        "gc_list_triangles": ([_vp, _vp, _i64, ctypes.POINTER(_i64)], ctypes.c_int),
        "gc_set_option": ([_vp, ctypes.c_int, _i64], ctypes.c_int),
        "gc_get_stats": ([_vp, ctypes.POINTER(gc_stats)], ctypes.c_int),
        "gc_reset_stats": ([_vp], ctypes.c_int),
        "gc_partition_bounds": ([_vp, _i64, ctypes.c_int, _vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _LIB = L
    return L


def __getattr__(name):  # module-level gc_* names resolve to the C entry points
    if name.startswith("gc_") and name in EXPORTS:
        return getattr(load_library(), name)
    raise AttributeError(name)


def _ptr(a) -> int:
    """Address of a numpy array or torch tensor (host or CUDA), contiguous."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported buffer type {type(a)}")


def _as_i32(a):
    if isinstance(a, np.ndarray) or not hasattr(a, "data_ptr"):
        return np.ascontiguousarray(a, dtype=np.int32)
    import torch
    if a.dtype != torch.int32:
        raise TypeError("edge tensors must be int32")
    return a.contiguous()


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = load_library().gc_nccl_unique_id(ctypes.cast(buf, _vp))
    if rc != GC_OK:
        raise GcError(rc, "gc_nccl_unique_id failed (NCCL unavailable?)")
    return buf.raw


class Context:
    """One libgc context on one GPU (see include/gc.h for every contract)."""

    def __init__(self, device: int = 0, stream=None):
        self._L = load_library()
        h = _vp()
        s = 0
        if stream is not None:
            s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        rc = self._L.gc_create(ctypes.byref(h), int(device), _vp(s) if s else None)
        if rc != GC_OK:
            raise GcError(rc, self._L.gc_last_error(None).decode())
        self._h = h
        self._staged = None
        self._pending_out = None
        self.device = device
        self._keep = []

    # -------------------------------------------------------------- util --
    def _check(self, rc: int):
        if rc != GC_OK:
            raise GcError(rc, self._L.gc_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.gc_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- calls --
    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        self._check(self._L.gc_comm_init(self._h, ctypes.cast(buf, _vp), int(nranks), int(rank)))

    def comm_init_loopback(self, nparts: int):
        self._check(self._L.gc_comm_init_loopback(self._h, int(nparts)))

    def load_edges(self, u, v):
        u = _as_i32(u)
        v = _as_i32(v)
        n = int(u.shape[0])
        if int(v.shape[0]) != n:
            raise ValueError("u and v differ in length")
        self._check(self._L.gc_load_edges(self._h, _vp(_ptr(u)), _vp(_ptr(v)), n))

    def stage_edges(self, u, v):
        """gc_stage_edges: start copying the next graph's raw list while the
        current one is in use; the next build_csr consumes it.  The arrays are
        kept referenced until then (page-locked host or device memory overlaps
        the copy with the kernels)."""
        u = _as_i32(u)
        v = _as_i32(v)
        n = int(u.shape[0])
        if int(v.shape[0]) != n:
            raise ValueError("u and v differ in length")
        self._check(self._L.gc_stage_edges(self._h, _vp(_ptr(u)), _vp(_ptr(v)), n))
        self._staged = (u, v)

    def build_csr(self):
        self._check(self._L.gc_build_csr(self._h))
        self._staged = None

    def num_vertices(self) -> int:
        x = _i64()
        self._check(self._L.gc_num_vertices(self._h, ctypes.byref(x)))
        return x.value

    def num_edges(self) -> int:
        x = _i64()
        self._check(self._L.gc_num_edges(self._h, ctypes.byref(x)))
        return x.value

    def get_edges(self, out_u=None, out_v=None):
        m = self.num_edges()
        if out_u is None:
            out_u = np.empty(m, dtype=np.int32)
        if out_v is None:
            out_v = np.empty(m, dtype=np.int32)
        self._check(self._L.gc_get_edges(self._h, _vp(_ptr(out_u)), _vp(_ptr(out_v))))
        return out_u, out_v

    def triangle_count(self) -> int:
        x = ctypes.c_uint64()
        self._check(self._L.gc_triangle_count(self._h, ctypes.byref(x)))
        return int(x.value)

    def edge_support(self, out=None):
        if out is None:
            out = np.empty(self.num_edges(), dtype=np.uint32)
        self._check(self._L.gc_edge_support(self._h, _vp(_ptr(out))))
        return out

    def ktruss(self, k: int, out=None):
        if out is None:
            out = np.empty(self.num_edges(), dtype=np.uint8)
        ma = _i64()
        self._check(self._L.gc_ktruss(self._h, int(k), _vp(_ptr(out)), ctypes.byref(ma)))
        return out, int(ma.value)

    def ktruss_analysis(self, k: int, support_out=None, mask_out=None):
        """Triangle count, per-edge support and the k-truss mask from one support pass
        (gc_ktruss_analysis).  Returns (triangles, support, mask, m_alive)."""
        m = self.num_edges()
        if support_out is None:
            support_out = np.empty(m, dtype=np.uint32)
        if mask_out is None:
            mask_out = np.empty(m, dtype=np.uint8)
        t = ctypes.c_uint64()
        ma = _i64()
        self._check(self._L.gc_ktruss_analysis(self._h, int(k), ctypes.byref(t), _vp(_ptr(support_out)),
                                               _vp(_ptr(mask_out)), ctypes.byref(ma)))
        return int(t.value), support_out, mask_out, int(ma.value)

    def ktruss_analysis_async(self, k: int, support_out, mask_out):
        """gc_ktruss_analysis_async: as ktruss_analysis into caller buffers
        (page-locked host or device) whose contents are valid only after
        wait().  Returns (triangles, m_alive) at once."""
        t = ctypes.c_uint64()
        ma = _i64()
        self._check(self._L.gc_ktruss_analysis_async(self._h, int(k), ctypes.byref(t), _vp(_ptr(support_out)),
                                                     _vp(_ptr(mask_out)), ctypes.byref(ma)))
        self._pending_out = (support_out, mask_out)
        return int(t.value), int(ma.value)

    def wait(self):
        """gc_wait: every asynchronous copy of this context is done."""
        self._check(self._L.gc_wait(self._h))
        self._pending_out = None

    def truss_decomposition(self, out=None):
        if out is None:
            out = np.empty(self.num_edges(), dtype=np.int32)
        km = _i32()
        self._check(self._L.gc_truss_decomposition(self._h, _vp(_ptr(out)), ctypes.byref(km)))
        return out, int(km.value)

    def list_triangles(self, capacity: int | None = None):
        """All triangles as an int32 array [T, 3] of original ids (ascending within
        a row; rows in unspecified order) -- gc_list_triangles."""
        cnt = _i64()
        if capacity is None:
            capacity = self.triangle_count()
        out = np.empty((max(int(capacity), 1), 3), dtype=np.int32)
        self._check(self._L.gc_list_triangles(self._h, _vp(_ptr(out)), int(capacity), ctypes.byref(cnt)))
        return out[:cnt.value]

    def set_option(self, option: int, value: int):
        self._check(self._L.gc_set_option(self._h, int(option), int(value)))

    def stats(self) -> dict:
        s = gc_stats()
        self._check(self._L.gc_get_stats(self._h, ctypes.byref(s)))
        out = {name: getattr(s, name) for name, _ in gc_stats._fields_}
        out["tasks"] = list(out["tasks"])
        out["aux"] = list(out["aux"])
        out["part_ms"] = list(out["part_ms"])
        out["part_build_ms"] = list(out["part_build_ms"])
        return out

    def reset_stats(self):
        self._check(self._L.gc_reset_stats(self._h))


def partition_bounds(cost_prefix, nparts: int) -> np.ndarray:
    """Host-side 1D owner cut (gc_partition_bounds): owner r holds [b[r], b[r+1])."""
    pref = np.ascontiguousarray(cost_prefix, dtype=np.int64)
    out = np.zeros(int(nparts) + 1, dtype=np.int64)
    rc = load_library().gc_partition_bounds(_vp(pref.ctypes.data), pref.size - 1, int(nparts),
                                             _vp(out.ctypes.data))
    if rc != GC_OK:
        raise GcError(rc, "gc_partition_bounds: bad arguments")
    return out


def init_distributed(ctx: Context, group=None):
    """Join ctx to an NCCL communicator spanning the torch.distributed world.

    Rank 0 draws the ncclUniqueId through libgc; torch.distributed (any
    backend) broadcasts the 128 bytes; every rank calls gc_comm_init."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if world == 1:
        return
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.comm_init(obj[0], world, rank)
