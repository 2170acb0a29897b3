"""Graph Challenge file formats (§II "Data Sets"): host-side
ingest into the int32 (u, v) pairs gc_load_edges takes.

* TSV: one edge per line, ``u<TAB>v<TAB>1``, vertices numbered 1..n.
* MMIO coordinate format (Matrix Market): ``%%MatrixMarket matrix
  coordinate ...`` header, ``%`` comments, a size line ``rows cols nnz``, then
  ``i j [value]`` lines, 1-based.

Ids are shifted to 0-based here, at the file boundary (reading D7 in SURVEY §8(b)).
Weights are ignored (all 1).  Self loops, duplicates and both
orientations are left in the pairs: gc_build_csr normalises them.
This module only parses text; no step of the method runs here.
"""
from __future__ import annotations

import numpy as np


def _pairs(cols0: np.ndarray, cols1: np.ndarray, what: str):
    u = cols0.astype(np.int64) - 1
    v = cols1.astype(np.int64) - 1
    if u.size and (min(u.min(), v.min()) < 0 or max(u.max(), v.max()) >= 2**31 - 1):
        raise ValueError(f"{what}: vertex ids must be in 1..2^31-1")
    return u.astype(np.int32), v.astype(np.int32)


def read_tsv(path: str):
    """Edge triples ``u v w`` (tab or space separated, 1-based) -> 0-based int32 (u, v)."""
    import pandas as pd
    df = pd.read_csv(path, sep=r"\s+", header=None, comment="#", dtype=np.int64, engine="c",
                     usecols=[0, 1])
    return _pairs(df[0].to_numpy(), df[1].to_numpy(), "read_tsv")


def write_tsv(path: str, u, v):
    """Inverse of read_tsv: 1-based ``u<TAB>v<TAB>1`` lines (the Graph Challenge layout)."""
    u = np.asarray(u, dtype=np.int64) + 1
    v = np.asarray(v, dtype=np.int64) + 1
    np.savetxt(path, np.stack([u, v, np.ones_like(u)], axis=1), fmt="%d", delimiter="\t")


def read_mmio(path: str):
    """Matrix Market coordinate file (pattern / integer / real; general or symmetric) -> 0-based (u, v)."""
    import pandas as pd
    with open(path) as f:
        header = f.readline()
        if not header.startswith("%%MatrixMarket") or "coordinate" not in header:
            raise ValueError("read_mmio: not a Matrix Market coordinate file")
        skip = 1
        line = f.readline()
        while line.startswith("%"):
            skip += 1
            line = f.readline()
        rows, cols, nnz = (int(x) for x in line.split()[:3])
        skip += 1
    if nnz == 0:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    df = pd.read_csv(path, sep=r"\s+", header=None, skiprows=skip, comment="%", usecols=[0, 1], dtype=np.int64,
                     engine="c")
    if len(df) != nnz:
        raise ValueError(f"read_mmio: {len(df)} entries, header says {nnz}")
    return _pairs(df[0].to_numpy(), df[1].to_numpy(), "read_mmio")


def write_mmio(path: str, u, v, n: int | None = None):
    """Pattern general coordinate file, 1-based."""
    u = np.asarray(u, dtype=np.int64) + 1
    v = np.asarray(v, dtype=np.int64) + 1
    if n is None:
        n = int(max(u.max(initial=0), v.max(initial=0)))
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate pattern general\n")
        f.write(f"{n} {n} {u.size}\n")
        np.savetxt(f, np.stack([u, v], axis=1), fmt="%d", delimiter=" ")
