"""CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_1708_06866_b200``) never imports it; the two share no code — only the
seeded generators in ``gen/`` serve both.

Thin ctypes wrapper over ``oracle/liboracle.so`` (oracle/oracle.c, plain C).
Each method names the PAPER.md passage it follows; see oracle.c's header.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

i32p = ctypes.POINTER(ctypes.c_int32)
i64p = ctypes.POINTER(ctypes.c_int64)
u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)
u8p = ctypes.POINTER(ctypes.c_uint8)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} oracle`")
        L = ctypes.CDLL(path)
        L.or_sort_u64.argtypes = [u64p, ctypes.c_int64]
        L.or_sort_u64.restype = ctypes.c_int
        L.or_canonicalize.argtypes = [i32p, i32p, ctypes.c_int64, i32p, i32p, i64p]
        L.or_canonicalize.restype = ctypes.c_int64
        L.or_adjacency.argtypes = [ctypes.c_int64, ctypes.c_int64, i32p, i32p, i64p, i32p, i32p]
        L.or_adjacency.restype = None
        L.or_support.argtypes = [i64p, i32p, ctypes.c_int64, i32p, i32p, u32p, ctypes.c_int]
        L.or_support.restype = None
        L.or_triangle_count.argtypes = [i64p, i32p, ctypes.c_int64, i32p, i32p, ctypes.c_int]
        L.or_triangle_count.restype = ctypes.c_uint64
        L.or_ktruss.argtypes = [ctypes.c_int64, ctypes.c_int64, i32p, i32p, i64p, i32p, i32p,
                                ctypes.c_int32, u8p, i64p, ctypes.c_int64, ctypes.c_int, i64p]
        L.or_ktruss.restype = ctypes.c_int64
        L.or_truss_decomposition.argtypes = [ctypes.c_int64, ctypes.c_int64, i32p, i32p, i64p, i32p,
                                             i32p, i32p, i32p, ctypes.c_int, i64p]
        L.or_truss_decomposition.restype = ctypes.c_int64
        L.or_truss_sequential.argtypes = [ctypes.c_int64, ctypes.c_int64, i32p, i32p, i64p, i32p,
                                          i32p, u32p, i32p, i32p, ctypes.c_int]
        L.or_truss_sequential.restype = ctypes.c_int64
        L.or_truss_parallel.argtypes = [ctypes.c_int64, ctypes.c_int64, i32p, i32p, i64p, i32p, i32p, u32p,
                                        i32p, i32p, ctypes.c_int]
        L.or_truss_parallel.restype = ctypes.c_int64
        L.or_truss_parallel_ckpt.argtypes = [ctypes.c_int64, ctypes.c_int64, i32p, i32p, i64p, i32p, i32p, u32p,
                                             i32p, i32p, ctypes.c_int, ctypes.c_char_p, ctypes.c_double]
        L.or_truss_parallel_ckpt.restype = ctypes.c_int64
        _LIB = L
    return _LIB


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def sort_u64(keys: np.ndarray) -> np.ndarray:
    k = np.ascontiguousarray(keys, dtype=np.uint64).copy()
    if _lib().or_sort_u64(_p(k, u64p), k.size) != 0:
        raise MemoryError
    return k


class OracleGraph:
    """Canonical graph + sorted adjacency built by the oracle from raw pairs."""

    def __init__(self, u, v, nthreads: int = 0):
        u = np.ascontiguousarray(u, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.int32)
        if u.shape != v.shape:
            raise ValueError("u and v differ in length")
        L = _lib()
        nnz = u.size
        cu = np.empty(max(nnz, 1), dtype=np.int32)
        cv = np.empty(max(nnz, 1), dtype=np.int32)
        n = ctypes.c_int64(0)
        m = L.or_canonicalize(_p(u, i32p), _p(v, i32p), nnz, _p(cu, i32p), _p(cv, i32p), ctypes.byref(n))
        if m < 0:
            raise ValueError("negative vertex id (or out of memory)")
        self.n = int(n.value)
        self.m = int(m)
        self.cu = cu[: self.m].copy()
        self.cv = cv[: self.m].copy()
        self.ptr = np.zeros(self.n + 1, dtype=np.int64)
        self.col = np.empty(max(2 * self.m, 1), dtype=np.int32)
        self.eid = np.empty(max(2 * self.m, 1), dtype=np.int32)
        L.or_adjacency(self.n, self.m, _p(self.cu, i32p), _p(self.cv, i32p), _p(self.ptr, i64p),
                       _p(self.col, i32p), _p(self.eid, i32p))
        self.nthreads = nthreads

    # O-3
    def support(self) -> np.ndarray:
        return self.support_pairs(self.cu, self.cv)

    def support_pairs(self, a, b) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.int32)
        b = np.ascontiguousarray(b, dtype=np.int32)
        out = np.zeros(a.size, dtype=np.uint32)
        _lib().or_support(_p(self.ptr, i64p), _p(self.col, i32p), a.size, _p(a, i32p), _p(b, i32p),
                          _p(out, u32p), self.nthreads)
        return out

    # O-4
    def triangle_count(self) -> int:
        return int(_lib().or_triangle_count(_p(self.ptr, i64p), _p(self.col, i32p), self.m,
                                            _p(self.cu, i32p), _p(self.cv, i32p), self.nthreads))

    # O-5
    def ktruss(self, k: int, trace_cap: int = 1 << 16, work: bool = False):
        """(alive mask, |x| per round); work=True adds {"sum_min", "decrements"}:
        the k-truss byte model's terms over the batch rounds (oracle.c peel_batch)."""
        alive = np.zeros(max(self.m, 1), dtype=np.uint8)
        trace = np.zeros(trace_cap, dtype=np.int64)
        w = np.zeros(2, dtype=np.int64)
        r = _lib().or_ktruss(self.n, self.m, _p(self.cu, i32p), _p(self.cv, i32p), _p(self.ptr, i64p),
                             _p(self.col, i32p), _p(self.eid, i32p), int(k), _p(alive, u8p),
                             _p(trace, i64p), trace_cap, self.nthreads, _p(w, i64p) if work else None)
        if r < 0:
            raise ValueError("k must be >= 2")
        out = (alive[: self.m].copy(), trace[: min(r, trace_cap)].copy())
        if work:
            return out + ({"sum_min": int(w[0]), "decrements": int(w[1])},)
        return out

    # O-6
    def truss_decomposition(self, work: bool = False):
        tau = np.zeros(max(self.m, 1), dtype=np.int32)
        kmax = ctypes.c_int32(0)
        w = np.zeros(2, dtype=np.int64)
        _lib().or_truss_decomposition(self.n, self.m, _p(self.cu, i32p), _p(self.cv, i32p),
                                      _p(self.ptr, i64p), _p(self.col, i32p), _p(self.eid, i32p),
                                      _p(tau, i32p), ctypes.byref(kmax), self.nthreads,
                                      _p(w, i64p) if work else None)
        if work:
            return tau[: self.m].copy(), int(kmax.value), {"sum_min": int(w[0]), "decrements": int(w[1])}
        return tau[: self.m].copy(), int(kmax.value)

    # O-7
    def truss_sequential(self, support: np.ndarray | None = None, consume: bool = False):
        """O-7.  consume=True lets the peel use this graph's adjacency rows as
        its live-row storage (no copy; the graph is unusable afterwards)."""
        if support is None:
            support = self.support()
        support = np.ascontiguousarray(support, dtype=np.uint32)
        tau = np.zeros(max(self.m, 1), dtype=np.int32)
        kmax = ctypes.c_int32(0)
        r = _lib().or_truss_sequential(self.n, self.m, _p(self.cu, i32p), _p(self.cv, i32p),
                                       _p(self.ptr, i64p), _p(self.col, i32p), _p(self.eid, i32p),
                                       _p(support, u32p), _p(tau, i32p), ctypes.byref(kmax),
                                       1 if consume else 0)
        if r < 0:
            raise MemoryError("or_truss_sequential: out of memory (or m > 2^31-1)")
        if consume:
            self.col = self.eid = None
        return tau[: self.m].copy(), int(kmax.value)

    # O-8
    def truss_parallel(self, support: np.ndarray | None = None, consume: bool = False, ckpt: str | None = None,
                       budget_s: float = 0.0):
        """O-8: Alg. 4's incremental update element-wise, rounds parallel over
        the removed edges.  Uses the adjacency rows as scratch (copied unless
        consume=True, which leaves this graph unusable).  ckpt: resume from
        that file if it exists; with budget_s > 0 the run saves its state
        there at a level start once budget_s seconds have passed (after at
        least one level) and returns None (call again to continue)."""
        if support is None:
            support = self.support()
        support = np.ascontiguousarray(support, dtype=np.uint32)
        col, eid = (self.col, self.eid) if consume else (self.col.copy(), self.eid.copy())
        tau = np.zeros(max(self.m, 1), dtype=np.int32)
        kmax = ctypes.c_int32(0)
        r = _lib().or_truss_parallel_ckpt(self.n, self.m, _p(self.cu, i32p), _p(self.cv, i32p),
                                          _p(self.ptr, i64p), _p(col, i32p), _p(eid, i32p), _p(support, u32p),
                                          _p(tau, i32p), ctypes.byref(kmax), self.nthreads,
                                          ckpt.encode() if ckpt else None, float(budget_s))
        if consume:
            self.col = self.eid = None
        if r == -2:
            return None                                   # saved to ckpt, unfinished
        if r == -3:
            raise ValueError(f"or_truss_parallel: unreadable checkpoint {ckpt}")
        if r == -4:
            raise OSError(f"or_truss_parallel: could not write checkpoint {ckpt}")
        if r < 0:
            raise MemoryError("or_truss_parallel: out of memory (or m > 2^31-1)")
        return tau[: self.m].copy(), int(kmax.value)
