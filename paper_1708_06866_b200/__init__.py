"""B200-native per-edge triangle support, triangle counting and k-truss.

Samsi et al., "Static Graph Challenge: Subgraph Isomorphism" (arXiv
1708.06866).  The product is libgc.so (CUDA, sm_100a) behind the C ABI in
include/gc.h; ``gc`` is its thin ctypes binding.
"""
from .gc import (  # noqa: F401
    EXPORTS,
    GC_OPT_FORCE_CLASS,
    GC_OPT_TASK_CHUNK,
    GC_OPT_TIMING,
    GC_OPT_BLOCK_BITMAP,
    Context,
    GcError,
    init_distributed,
    load_library,
    nccl_unique_id,
)
from .io import read_mmio, read_tsv, write_mmio, write_tsv  # noqa: F401

__all__ = ["Context", "GcError", "init_distributed", "load_library", "nccl_unique_id", "EXPORTS"]
