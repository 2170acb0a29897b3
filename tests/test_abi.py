"""The C-ABI library loads and exports every symbol include/gc.h declares
(CPU only: no compute call is made without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gc.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gc_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ["gc_load_edges", "gc_build_csr", "gc_triangle_count", "gc_edge_support", "gc_ktruss"]:
        assert name in syms


def test_library_exports_every_declared_symbol(gc_lib_path):
    lib = ctypes.CDLL(gc_lib_path)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_binding_lists_every_declared_symbol():
    from paper_1708_06866_b200 import gc
    assert sorted(gc.EXPORTS) == declared_symbols()


def test_library_links_no_oracle(gc_lib_path):
    """The product library must not depend on the oracle (shares no code)."""
    data = open(gc_lib_path, "rb").read()
    assert b"or_support" not in data and b"liboracle" not in data and b"or_canonicalize" not in data


def test_create_without_gpu_fails_cleanly(gc_lib_path):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present; covered by the gpu tests")
    from paper_1708_06866_b200 import gc
    with pytest.raises(gc.GcError):
        gc.Context(0)


def test_null_context_calls_are_rejected(gc_lib_path):
    from paper_1708_06866_b200 import gc
    L = gc.load_library()
    x = ctypes.c_int64()
    assert L.gc_num_edges(None, ctypes.byref(x)) == gc.GC_ERR_INVALID
    assert L.gc_build_csr(None) == gc.GC_ERR_INVALID
    assert L.gc_destroy(None) == gc.GC_OK
