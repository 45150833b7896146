"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds none of the method's arithmetic: it draws M, X_L, y and the
X_R genotype columns of BASELINE.json `configs` (recipe in DESIGN.md §"Inputs" and
SURVEY.md §8(d)) with a counter-based Philox4x32-10 generator implemented in
`glsgen.c`.  The GPU genotype generator (paper_1210_7325_b200/csrc/gen_device.cu)
implements the same generator independently;
`tests/test_gpu_parity.py::test_device_generator_matches_cpu` checks the two agree bit
for bit.

Array conventions (column-major, as the C ABI): an n x k column-major matrix is a
C-contiguous numpy array of shape (k, n) -- row j of the array is column j.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "glsgen.c")
_LIB = os.path.join(_HERE, "libglsgen.so")

DEFAULT_SEED = 12107325


def build(force: bool = False) -> str:
    """Compile glsgen.c into gen/libglsgen.so (gcc, OpenMP, no FP contraction)."""
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
        u64, i64, i32, u32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
        dp = ctypes.POINTER(ctypes.c_double)
        L.glsgen_philox.argtypes = [u64, u32, u64, u32, ctypes.POINTER(ctypes.c_uint32)]
        L.glsgen_normals.argtypes = [u64, u32, u64, i64, dp]
        L.glsgen_q.argtypes = [u64, u64]
        L.glsgen_q.restype = ctypes.c_double
        L.glsgen_xr.argtypes = [u64, i64, u64, i64, dp, i64]
        L.glsgen_M.argtypes = [u64, i64, dp]
        L.glsgen_xl.argtypes = [u64, i64, i32, i32, dp]
        L.glsgen_y.argtypes = [u64, i64, i32, dp, ctypes.c_double, dp, dp]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# --------------------------------------------------------------------------- configs
@dataclass(frozen=True)
class Config:
    """One BASELINE.json `configs` entry (index `idx`)."""
    idx: int
    n: int
    pL: int
    pR: int
    m: int              # number of SNP groups (problems)
    with_sex: bool
    desc: str

    @property
    def p(self) -> int:
        return self.pL + self.pR

    @property
    def cols(self) -> int:
        return self.m * self.pR


CONFIGS = {
    0: Config(0, 500, 3, 1, 2000, True, "n=500 p=4 m=2000 (parity case)"),
    1: Config(1, 1500, 3, 1, 220_833, True, "n=1500 p=4 m=220833 (cited study shape)"),
    2: Config(2, 10_000, 3, 1, 1_000_000, True, "n=1e4 p=4 m=1e6 in-core (headline metric)"),
    3: Config(3, 10_000, 16, 4, 500_000, False, "n=1e4 pL=16 pR=4 m=5e5 groups"),
    4: Config(4, 10_000, 3, 1, 10_000_000, True, "n=1e4 p=4 m=1e7 out-of-core"),
}


def philox(seed: int, stream: int, index: int, sub: int = 0) -> np.ndarray:
    out = (ctypes.c_uint32 * 4)()
    lib().glsgen_philox(seed, stream, index, sub, out)
    return np.array(list(out), dtype=np.uint32)


def normals(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    lib().glsgen_normals(seed, stream, start, count, _dp(out))
    return out


def q_of(seed: int, col: int) -> float:
    return lib().glsgen_q(seed, col)


def make_M(seed: int, n: int) -> np.ndarray:
    """M = 0.5 Z Z^T / 256 + 0.5 I (symmetric; returned as an (n, n) array)."""
    M = np.empty((n, n), dtype=np.float64)
    lib().glsgen_M(seed, n, _dp(M))
    return M


def make_XL(seed: int, n: int, pL: int, with_sex: bool) -> np.ndarray:
    """X_L column-major: array of shape (pL, n)."""
    XL = np.empty((max(pL, 0), n), dtype=np.float64)
    if pL > 0:
        lib().glsgen_xl(seed, n, pL, 1 if with_sex else 0, _dp(XL))
    return XL


def make_y(seed: int, XL: np.ndarray, n: int, noise: float = 1.0):
    """y = X_L beta_L + noise * eps.  Returns (y, beta_L)."""
    pL = XL.shape[0]
    beta = np.empty(max(pL, 1), dtype=np.float64)
    y = np.empty(n, dtype=np.float64)
    xl = XL if pL > 0 else np.zeros((1, n))
    lib().glsgen_y(seed, n, pL, _dp(np.ascontiguousarray(xl)), float(noise), _dp(beta), _dp(y))
    return y, beta[:pL]


def make_XR(seed: int, n: int, col0: int, ncols: int, out: np.ndarray | None = None) -> np.ndarray:
    """Genotype columns [col0, col0+ncols) as a (ncols, n) array (column-major n x ncols)."""
    if out is None:
        out = np.empty((ncols, n), dtype=np.float64)
    assert out.shape == (ncols, n)
    if ncols > 0:
        lib().glsgen_xr(seed, n, col0, ncols, _dp(out), n)
    return out


@dataclass
class Problem:
    n: int
    pL: int
    pR: int
    M: np.ndarray        # (n, n) symmetric
    XL: np.ndarray       # (pL, n)  column-major n x pL
    y: np.ndarray        # (n,)
    beta_L: np.ndarray   # (pL,)


def make_problem(n: int, pL: int, pR: int, with_sex: bool = True, seed: int = DEFAULT_SEED,
                 noise: float = 1.0) -> Problem:
    M = make_M(seed, n)
    XL = make_XL(seed, n, pL, with_sex)
    y, beta = make_y(seed, XL, n, noise)
    return Problem(n, pL, pR, M, XL, y, beta)


def config_problem(cfg: Config, seed: int = DEFAULT_SEED, noise: float = 1.0) -> Problem:
    return make_problem(cfg.n, cfg.pL, cfg.pR, cfg.with_sex, seed, noise)
