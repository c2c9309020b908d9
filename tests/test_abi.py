"""Host-side checks of the C-ABI boundary (no GPU needed): the library loads, exports exactly the
symbols include/rg.h declares, and rejects invalid arguments before touching the device."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rg.h")
LIB = os.path.join(ROOT, "paper_1807_09467_b200", "lib", "librg.so")


def declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"RG_API\s+[\w\s\*]+?\b(rg_\w+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    d = declared()
    for f in ("rg_create", "rg_update_matrix", "rg_push_snapshot", "rg_build_recycle", "rg_solve",
              "rg_destroy", "rg_last_error"):
        assert f in d


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    d = set(declared())
    assert d <= exported, d - exported
    # nothing else leaks (hidden visibility): only rg_* API symbols are exported
    assert {s for s in exported if s.startswith("rg_")} == d


def test_binding_names_match_header():
    from paper_1807_09467_b200 import rg
    assert set(rg.SYMBOLS) == set(declared())
    for f in rg.SYMBOLS:
        assert callable(getattr(rg, f))


def test_create_rejects_invalid_arguments_without_device():
    from paper_1807_09467_b200 import rg
    rp = np.array([0, 1, 2], np.int32)
    ci = np.array([0, 1], np.int32)
    v = np.array([1.0, 1.0])
    good = rg.make_matrix(2, rp, ci, v)
    with pytest.raises(rg.RgError) as e:
        rg.rg_create(0, good)
    assert e.value.status == rg.RG_E_INVAL
    with pytest.raises(rg.RgError) as e:
        rg.rg_create(2, good, max_m=0)
    assert e.value.status == rg.RG_E_INVAL
    with pytest.raises(rg.RgError) as e:
        rg.rg_create(2, good, max_k=65)
    assert e.value.status == rg.RG_E_INVAL
    # n_rows mismatch (descriptor built by hand: make_matrix itself refuses the short row_ptr)
    bad = rg.rg_matrix(rg.RG_CSR, 3, 2, 1, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, rg.RG_HOST, 0, 1)
    with pytest.raises(rg.RgError) as e:
        rg.rg_create(2, bad)
    assert e.value.status == rg.RG_E_INVAL
    assert "n_rows" in rg.rg_last_error()


def test_null_context_is_inval():
    from paper_1807_09467_b200 import rg
    L = rg._lib
    assert L.rg_solve(None, None, None, 10, 0, 1e-8, 10, None, 0, None, 0, None) == rg.RG_E_INVAL
    assert L.rg_push_snapshot(None, None, 0) == rg.RG_E_INVAL
    L.rg_destroy(None)   # no-op


def test_oracle_library_is_separate():
    """The product library links no oracle code and the oracle links no CUDA."""
    out = subprocess.run(["nm", "-D", LIB], capture_output=True, text=True, check=True).stdout
    assert "or_solve" not in out and "or_svd" not in out
    olib = os.path.join(ROOT, "oracle", "liboracle.so")
    dep = subprocess.run(["ldd", olib], capture_output=True, text=True).stdout
    assert "cuda" not in dep


def test_binding_checks_dtype_and_length():
    """The binding refuses buffers the C ABI would read or write past (float32 / short
    vectors, int64 index arrays)."""
    from paper_1807_09467_b200 import rg
    rp = np.array([0, 1, 2], np.int32)
    ci = np.array([0, 1], np.int32)
    v = np.array([1.0, 1.0])
    with pytest.raises(ValueError):
        rg.make_matrix(3, rp, ci, v)                      # row_ptr shorter than n + 1
    with pytest.raises(TypeError):
        rg.make_matrix(2, rp.astype(np.int64), ci, v)     # int64 indices
    with pytest.raises(TypeError):
        rg.make_matrix(2, rp, ci, v.astype(np.float32))   # float32 values
    with pytest.raises(ValueError):
        rg.make_matrix(2, rp, ci[:1], v)                  # col_idx shorter than nnz
    rg._CTX_N[12345] = 10
    try:
        with pytest.raises(TypeError):
            rg.rg_solve(12345, np.zeros(10, np.float32), np.zeros(10))
        with pytest.raises(ValueError):
            rg.rg_solve(12345, np.zeros(10), np.zeros(9))
        with pytest.raises(ValueError):
            rg.rg_push_snapshot(12345, np.zeros(9))
    finally:
        rg._CTX_N.pop(12345)
