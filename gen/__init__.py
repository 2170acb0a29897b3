"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

Input harness only: this module emits raw directed pairs (u, v) and holds none
of the method's arithmetic.  The C implementation (gen/gen.c) is compiled to
``gen/libgcgen.so`` by ``make gen`` (or ``__graft_entry__.build()``).

Configs C1..C5 are BASELINE.json ``configs[0..4]`` (SURVEY.md §8 "Config
shorthand"); C1 is the small case the oracle finishes in seconds, C4 (R-MAT
scale 24) is the configuration the headline metric is quoted on.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libgcgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} gen`")
        L = ctypes.CDLL(path)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.gen_rmat.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_uint64, ctypes.c_int, i32p, i32p, ctypes.c_int]
        L.gen_rmat.restype = ctypes.c_int
        L.gen_er_count.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int]
        L.gen_er_count.restype = ctypes.c_int64
        L.gen_er_fill.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, i32p, i32p,
                                  ctypes.c_int64, ctypes.c_int]
        L.gen_er_fill.restype = ctypes.c_int64
        L.gen_king_grid.argtypes = [ctypes.c_int64, i32p, i32p]
        L.gen_king_grid.restype = ctypes.c_int64
        L.gen_hash.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        L.gen_hash.restype = ctypes.c_uint64
        L.gen_vertex_perm.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32]
        L.gen_vertex_perm.restype = ctypes.c_uint32
        _LIB = L
    return _LIB


def _p32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
         seed: int = 1, permute: bool = True, nthreads: int = 0):
    """Raw R-MAT pairs: nnz = edge_factor * 2**scale, self-loops/duplicates kept."""
    nnz = int(edge_factor) << int(scale)
    u = np.empty(nnz, dtype=np.int32)
    v = np.empty(nnz, dtype=np.int32)
    rc = _lib().gen_rmat(int(scale), nnz, float(a), float(b), float(c), int(seed) & (2**64 - 1),
                         1 if permute else 0, _p32(u), _p32(v), int(nthreads))
    if rc != 0:
        raise ValueError("gen_rmat: bad arguments")
    return u, v


def erdos_renyi(n: int, mean_degree: float = 32.0, seed: int = 2, nthreads: int = 0):
    """G(n, p) with p = mean_degree / (n - 1); each edge once, hashed orientation."""
    p = float(mean_degree) / float(n - 1) if n > 1 else 0.0
    L = _lib()
    cnt = L.gen_er_count(int(n), p, int(seed), int(nthreads))
    if cnt < 0:
        raise ValueError("gen_er_count: bad arguments")
    u = np.empty(cnt, dtype=np.int32)
    v = np.empty(cnt, dtype=np.int32)
    got = L.gen_er_fill(int(n), p, int(seed), _p32(u), _p32(v), cnt, int(nthreads))
    if got != cnt:
        raise RuntimeError("gen_er_fill: count mismatch")
    return u, v


def king_grid(M: int):
    """The paper's M x M image graph: 2(M-1)(2M-1) undirected pairs."""
    cap = max(0, 2 * (M - 1) * (2 * M - 1))
    u = np.empty(cap, dtype=np.int32)
    v = np.empty(cap, dtype=np.int32)
    k = _lib().gen_king_grid(int(M), _p32(u), _p32(v))
    return u[:k], v[:k]


def gen_hash(seed: int, a: int, b: int) -> int:
    return int(_lib().gen_hash(seed & (2**64 - 1), a & (2**64 - 1), b & (2**64 - 1)))


def vertex_perm(seed: int, s: int, x: int) -> int:
    return int(_lib().gen_vertex_perm(seed & (2**64 - 1), int(s), int(x)))


@dataclass(frozen=True)
class Config:
    name: str
    kind: str            # "rmat" | "er" | "king" (n = M, the grid side)
    scale: int = 0
    edge_factor: int = 16
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    seed: int = 1
    n: int = 0
    mean_degree: float = 0.0
    desc: str = ""

    def generate(self, nthreads: int = 0):
        if self.kind == "rmat":
            return rmat(self.scale, self.edge_factor, self.a, self.b, self.c, self.seed, True, nthreads)
        if self.kind == "er":
            return erdos_renyi(self.n, self.mean_degree, self.seed, nthreads)
        if self.kind == "king":
            return king_grid(self.n)
        raise ValueError(self.kind)


# BASELINE.json configs[0..4]
CONFIGS = {
    "C1": Config("C1", "rmat", scale=10, seed=1, desc="R-MAT s10 ef16 (0.57,0.19,0.19,0.05) seed 1"),
    "C2": Config("C2", "er", n=65536, mean_degree=32.0, seed=2, desc="ER n=65536 mean degree 32 seed 2"),
    "C3": Config("C3", "rmat", scale=20, seed=3, desc="R-MAT s20 ef16 (0.57,0.19,0.19,0.05) seed 3"),
    "C4": Config("C4", "rmat", scale=24, seed=4, desc="R-MAT s24 ef16 (0.57,0.19,0.19,0.05) seed 4"),
    "C5": Config("C5", "rmat", scale=26, a=0.65, b=0.15, c=0.15, seed=5,
                 desc="R-MAT s26 ef16 skewed (0.65,0.15,0.15,0.05) seed 5"),
    # the paper's own synthetic graphs, Table II: M x M king grids, M = 2^12, 2^13
    "K12": Config("K12", "king", n=4096, desc="king grid M=4096 (Table II row 12: 67,084,290 edges)"),
    "K13": Config("K13", "king", n=8192, desc="king grid M=8192 (Table II row 13: 268,386,306 edges)"),
}
