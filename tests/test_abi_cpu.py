"""CPU-side checks of the boundary: libgls.so loads and exports every symbol include/gls.h
declares; argument/dimension validation runs without touching the GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "gls.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gls_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1210_7325_b200 import gls
    return gls.load()


def test_header_declares_boundary():
    syms = header_symbols()
    for s in ("gls_create", "gls_solve_block", "gls_destroy"):
        assert s in syms


def test_library_exports_every_header_symbol(lib):
    from paper_1210_7325_b200 import gls
    syms = header_symbols()
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(gls.ABI_SYMBOLS) == syms


def test_error_strings(lib):
    for code in range(7):
        s = lib.gls_error_string(code).decode()
        assert s.startswith("GLS_")
    assert b"unknown" in lib.gls_error_string(99)


@pytest.mark.parametrize("n,pL,pR,code", [(10, 3, 0, 2), (4, 3, 1, 2), (100, -1, 1, 2),
                                           (100, 17, 4, 2), (100, 0, 21, 2), (21, 19, 1, 0)])
def test_dims_validated_before_device_work(lib, n, pL, pR, code):
    """GLS_ERR_DIM unless n > p, pL >= 0, pR >= 1, p <= 20."""
    h = ctypes.c_void_p(123)
    if code == 0:
        # valid dims but NULL M -> GLS_ERR_ARG, *out NULL, no CUDA call
        assert lib.gls_create(n, pL, pR, None, None, None, ctypes.byref(h)) == 1
        assert h.value is None
        return
    buf = (ctypes.c_double * 4)()
    rc = lib.gls_create(n, pL, pR, buf, buf, buf, ctypes.byref(h))
    assert rc == code and h.value is None
    assert lib.gls_create_adopt(n, pL, pR, ctypes.byref(h)) == code


def test_null_handles(lib):
    assert lib.gls_solve_block(None, None, 1, None) == 1
    assert lib.gls_sync(None) == 1
    assert lib.gls_failed_pivot(None) == -1
    assert lib.gls_last_error(None) == b""
    lib.gls_destroy(None)
    assert lib.gls_create(10, 1, 1, None, None, None, None) == 1


def test_null_handles_extensions(lib):
    i64 = ctypes.c_int64
    a, b = i64(), i64()
    assert lib.gls_set_path(None, 0) == 1
    assert lib.gls_path_counts(None, ctypes.byref(a), ctypes.byref(b)) == 1
    assert lib.gls_solve_block_i8(None, None, 10, 1, None, None, 0) == 1
    assert lib.gls_set_timing(None, 1) == 1
    d = ctypes.c_double()
    assert lib.gls_read_timing(None, ctypes.byref(d), ctypes.byref(d), ctypes.byref(d), ctypes.byref(a)) == 1
    assert lib.gls_set_stream_report(None, 1) == 1
    assert lib.gls_read_stream_report(None, None) == 1


def test_select_block_size_condition():
    """§4.3: time(compute) > time(load) + time(store); two workspaces in memory."""
    from paper_1210_7325_b200 import select_block_size
    n, p, pR = 10_000, 4, 1
    per = pR * n * 8 + p * 8 + 4
    # memory caps the block: two workspaces of k problems
    k, io = select_block_size(n, p, pR, 8, 2 * per * 1000, compute_groups_per_s=3e5, io_bytes_per_s=55e9)
    assert k == 1000
    # FP64 X_R over 55 GB/s: 80 kB per problem = 1.45 us of PCIe vs 3.3 us of compute -> compute-bound
    assert io is False
    # int8 codes at 3 M problems/s are compute-bound at 55 GB/s (10 kB per problem = 0.18 us vs 0.33 us)
    k8, io8 = select_block_size(n, p, pR, 1, 1 << 34, compute_groups_per_s=3e6, io_bytes_per_s=55e9)
    assert io8 is False and k8 == (1 << 34) // (2 * (n + p * 8 + 4))
    # FP64 X_R at 3 M problems/s over 55 GB/s is I/O-bound (the paper's n > 8 F / B condition fails)
    _, iob = select_block_size(n, p, pR, 8, 1 << 34, compute_groups_per_s=3e6, io_bytes_per_s=55e9)
    assert iob is True
    # a per-request latency makes small blocks I/O-bound
    _, iol = select_block_size(n, p, pR, 1, 2 * (n + 36) * 10, compute_groups_per_s=3e6, io_bytes_per_s=55e9,
                               io_latency_s=1e-3)
    assert iol is True
    assert select_block_size(n, p, pR, 3, 1 << 30, 1.0, 1.0)[0] == -1
    assert select_block_size(n, p, pR, 8, 10, 1.0, 1.0)[0] == -1
