"""CPU: libtrals.so loads and exports every entry point include/trals.h declares."""

import os
import re

from paper_2210_11362_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "trals.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(trals_[a-z0-9_]+)\s*\(", text))


def test_header_and_binding_agree():
    assert header_functions() == set(_lib.EXPORTED)


def test_library_exports_every_symbol():
    h = _lib.load()
    for name in header_functions():
        assert getattr(h, name) is not None
    assert h.trals_version() == 1
    assert h.trals_strerror(3) == b"workspace too small"


def test_workspace_queries_without_gpu():
    h = _lib.load()
    # ragged-wave fix: the c5 environment GEMM (1000 tiles on 296 slots) is split 5-way in K
    assert h.trals_gemm_ws_elems(1, 25600, 25600, 400) == 5 * 25600 * 400
    assert h.trals_gemm_ws_elems(1, 250000, 500, 100) == 0
    assert h.trals_gemm_ws_elems(1, 1600, 64000, 64) > 0      # long-K shapes split K deterministically
    dims = _lib.i64_array([160] * 4)
    ranks = _lib.i32_array([20] * 4)
    assert h.trals_mttsp_ws_elems(4, dims, ranks, 0) > 0
