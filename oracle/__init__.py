"""CPU FP64 oracle for the GLS sequence b_i = (X_i^T M^-1 X_i)^-1 X_i^T M^-1 y.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` leg may import this package.  The product path
(`paper_1210_7325_b200/`) never imports it, and the two share no code.

The arithmetic lives in `gls_oracle.c` (plain scalar loops, Alg. 4 seq-gls with
Alg. 3's per-problem steps; see its header for the passages followed).  This module
only compiles it with gcc and marshals numpy arrays through ctypes.

Pins (tests/test_oracle_pins.py) tie every function here to something other than
itself: SPEC/paper worked examples, exact-rational brute force, the M = I OLS closed
form, scaling invariance, the planted-beta identity, orthogonality and a LAPACK
cross-check.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gls_oracle.c")
_LIB = os.path.join(_HERE, "libgls_oracle.so")

ORACLE_OK = 0
ORACLE_NOT_SPD = 3


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC",
                               "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_cholesky.argtypes = [i64, dp, i64, dp, ctypes.POINTER(ctypes.c_int64)]
        L.oracle_cholesky.restype = ctypes.c_int
        L.oracle_forward.argtypes = [i64, dp, dp, dp]
        L.oracle_spd_solve.argtypes = [i32, dp, dp, dp]
        L.oracle_spd_solve.restype = ctypes.c_int
        L.oracle_gls_sequence.argtypes = [i64, i32, i32, dp, dp, dp, dp, i64, i32, i64,
                                          ctypes.POINTER(ctypes.c_int64), dp,
                                          ctypes.POINTER(ctypes.c_int32)]
        _lib = L
    return _lib


def _dp(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class NotSPD(Exception):
    def __init__(self, pivot: int):
        super().__init__("M is not SPD: pivot %d" % pivot)
        self.pivot = pivot


def cholesky(M: np.ndarray) -> np.ndarray:
    """L (row-major lower, as an (n, n) array L[i, k]) with L L^T = M.  Raises NotSPD."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    n = M.shape[0]
    # M symmetric: its C-order buffer read column-major is M^T = M; lower triangle of
    # the column-major view is what the C code reads.
    Mc = np.ascontiguousarray(M.T)
    L = np.empty((n, n), dtype=np.float64)
    piv = ctypes.c_int64(-1)
    rc = lib().oracle_cholesky(n, _dp(Mc), n, _dp(L), ctypes.byref(piv))
    if rc != ORACLE_OK:
        raise NotSPD(piv.value)
    return L


def forward(L: np.ndarray, b: np.ndarray) -> np.ndarray:
    """x with L x = b (L row-major lower as returned by cholesky)."""
    n = L.shape[0]
    x = np.empty(n, dtype=np.float64)
    lib().oracle_forward(n, _dp(np.ascontiguousarray(L)), _dp(np.ascontiguousarray(b, dtype=np.float64)), _dp(x))
    return x


def spd_solve(S: np.ndarray, r: np.ndarray):
    """(b, status) for S b = r, S p x p SPD (lower triangle read).  status 1 = RankDeficient."""
    S = np.asarray(S, dtype=np.float64)
    p = S.shape[0]
    Sc = np.ascontiguousarray(S.T)  # column-major buffer
    b = np.empty(p, dtype=np.float64)
    st = lib().oracle_spd_solve(p, _dp(Sc), _dp(np.ascontiguousarray(r, dtype=np.float64)), _dp(b))
    return b, int(st)


def gls_sequence(L: np.ndarray, XL: np.ndarray, y: np.ndarray, XR: np.ndarray, pR: int,
                 sel=None, xr_is_selected: bool = False):
    """b rows and status for the problems in `sel` (default: all).

    L:  (n, n) row-major lower factor from `cholesky`.
    XL: (pL, n) -- X_L column-major.   y: (n,).
    XR: (ncols, n) -- X_R column-major; problem i uses columns [i*pR, (i+1)*pR), or
        [t*pR, (t+1)*pR) for the t-th selected problem when xr_is_selected.
    Returns (b, status): b (nsel, p), status (nsel,) int32.
    """
    n = L.shape[0]
    pL = XL.shape[0]
    p = pL + pR
    XR = np.ascontiguousarray(XR, dtype=np.float64)
    if sel is None:
        sel = np.arange(XR.shape[0] // pR, dtype=np.int64)
    sel = np.ascontiguousarray(sel, dtype=np.int64)
    nsel = sel.shape[0]
    b = np.empty((nsel, p), dtype=np.float64)
    st = np.empty(nsel, dtype=np.int32)
    xl = np.ascontiguousarray(XL, dtype=np.float64) if pL > 0 else np.zeros((1, n))
    lib().oracle_gls_sequence(n, pL, pR, _dp(np.ascontiguousarray(L)), _dp(xl),
                              _dp(np.ascontiguousarray(y, dtype=np.float64)), _dp(XR), n,
                              1 if xr_is_selected else 0, nsel,
                              sel.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(b),
                              st.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return b, st


def solve(M, XL, y, XR, pR: int, sel=None, xr_is_selected: bool = False):
    """Full oracle: Cholesky of M then the sequence.  Returns (b, status)."""
    L = cholesky(M)
    return gls_sequence(L, XL, y, XR, pR, sel, xr_is_selected)
