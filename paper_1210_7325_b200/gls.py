"""Thin ctypes binding of libgls.so (include/gls.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels.  There is no CPU fallback:
if libgls.so is missing or no CUDA device is present, calls raise GLSError.

Array arguments may be torch tensors (CPU, pinned CPU or CUDA; float64 / int32, contiguous)
or numpy arrays (host).  Column-major n x k matrices are passed as contiguous arrays of
shape (k, n): row j of the array is column j of the matrix.
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

GLS_OK = 0
GLS_ERR_ARG = 1
GLS_ERR_DIM = 2
GLS_ERR_NOT_SPD = 3
GLS_ERR_CUDA = 4
GLS_ERR_OOM = 5
GLS_ERR_STATE = 6
GLS_PATH_AUTO = 0
GLS_PATH_FP64 = 1
GLS_OOC_SYNC = 0
GLS_OOC_ASYNC = 1
GLS_GWFGLS_GEMV = 0
GLS_GWFGLS_GEMM = 1
GLS_SHARE_INT8_ONLY = 1
GLS_DIST_FACTOR, GLS_DIST_UPDATE, GLS_DIST_PARTIALS, GLS_DIST_PACK, GLS_DIST_PACK2 = range(5)
GLS_DIST_PANEL, GLS_DIST_WPART, GLS_DIST_W, GLS_DIST_ROWMAX, GLS_DIST_VMAX, GLS_DIST_T8, GLS_DIST_V8 = range(7)


class OocReport(ctypes.Structure):
    """gls_ooc_report: wait times at the wait points of Alg. 7 / Alg. 8."""
    _fields_ = [("wall_s", ctypes.c_double), ("compute_s", ctypes.c_double), ("read_wait_s", ctypes.c_double),
                ("write_wait_s", ctypes.c_double), ("first_load_s", ctypes.c_double),
                ("blocks", ctypes.c_int64), ("bytes_read", ctypes.c_int64), ("bytes_written", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class StreamReport(ctypes.Structure):
    """gls_stream_report: overlap accounting of the host -> HBM stream (Alg. 8)."""
    _fields_ = [("chunks", ctypes.c_int64), ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
                ("wall_ms", ctypes.c_double), ("h2d_ms", ctypes.c_double), ("compute_ms", ctypes.c_double),
                ("d2h_ms", ctypes.c_double), ("first_load_ms", ctypes.c_double),
                ("exposed_h2d_ms", ctypes.c_double), ("exposed_other_ms", ctypes.c_double),
                ("tail_ms", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}

ABI_SYMBOLS = (
    "gls_create", "gls_create_async", "gls_solve_block", "gls_solve_block_ex", "gls_sync", "gls_set_stream",
    "gls_set_block_cols", "gls_destroy", "gls_failed_pivot", "gls_last_error",
    "gls_error_string", "gls_create_adopt", "gls_shared_view", "gls_commit_shared",
    "gls_kernel_launches", "gls_set_path", "gls_path_counts", "gls_solve_block_i8",
    "gls_set_timing", "gls_read_timing", "gls_get_dims", "gls_solve_file", "gls_select_block_size",
    "gls_release_cached_memory", "gls_set_stream_report", "gls_read_stream_report",
    "gls_gwfgls_create", "gls_gwfgls_solve", "gls_gwfgls_launches", "gls_gwfgls_destroy",
    "gls_create_adopt_int8", "gls_shared_view_ex",
    "gls_dist_create", "gls_dist_info", "gls_dist_buffer", "gls_dist_step", "gls_dist_finish",
    "gls_dist_failed_pivot", "gls_dist_launches", "gls_dist_destroy",
)


class GLSError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


_lib = None
_gen = None


def load(build_if_missing: bool = True):
    """Load libgls.so (building it in-tree with nvcc if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.lib_path("libgls.so")
    if not os.path.exists(path) and build_if_missing:
        _build.build()
    if not os.path.exists(path):
        raise GLSError(GLS_ERR_CUDA, "libgls.so not built (python -m paper_1210_7325_b200.build)")
    L = ctypes.CDLL(path)
    vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    L.gls_create.argtypes = [i64, i32, i32, dp, dp, dp, ctypes.POINTER(vp)]
    L.gls_create.restype = ctypes.c_int
    L.gls_create_async.argtypes = [i64, i32, i32, dp, dp, dp, ctypes.POINTER(vp)]
    L.gls_create_async.restype = ctypes.c_int
    L.gls_create_adopt.argtypes = [i64, i32, i32, ctypes.POINTER(vp)]
    L.gls_create_adopt.restype = ctypes.c_int
    L.gls_solve_block.argtypes = [vp, dp, i64, dp]
    L.gls_solve_block.restype = ctypes.c_int
    L.gls_solve_block_ex.argtypes = [vp, dp, i64, dp, dp, ctypes.c_int]
    L.gls_solve_block_ex.restype = ctypes.c_int
    L.gls_sync.argtypes = [vp]
    L.gls_sync.restype = ctypes.c_int
    L.gls_set_stream.argtypes = [vp, vp]
    L.gls_set_stream.restype = ctypes.c_int
    L.gls_set_block_cols.argtypes = [vp, i64]
    L.gls_set_block_cols.restype = ctypes.c_int
    L.gls_destroy.argtypes = [vp]
    L.gls_destroy.restype = None
    L.gls_failed_pivot.argtypes = [vp]
    L.gls_failed_pivot.restype = i64
    L.gls_last_error.argtypes = [vp]
    L.gls_last_error.restype = ctypes.c_char_p
    L.gls_error_string.argtypes = [ctypes.c_int]
    L.gls_error_string.restype = ctypes.c_char_p
    L.gls_shared_view.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.gls_shared_view.restype = ctypes.c_int
    L.gls_commit_shared.argtypes = [vp]
    L.gls_commit_shared.restype = ctypes.c_int
    L.gls_kernel_launches.argtypes = [vp]
    L.gls_kernel_launches.restype = i64
    L.gls_set_path.argtypes = [vp, i32]
    L.gls_set_path.restype = ctypes.c_int
    L.gls_path_counts.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.gls_path_counts.restype = ctypes.c_int
    L.gls_solve_block_i8.argtypes = [vp, dp, i64, i64, dp, dp, ctypes.c_int]
    L.gls_solve_block_i8.restype = ctypes.c_int
    L.gls_set_timing.argtypes = [vp, i32]
    L.gls_set_timing.restype = ctypes.c_int
    dpp = ctypes.POINTER(ctypes.c_double)
    L.gls_read_timing.argtypes = [vp, dpp, dpp, dpp, ctypes.POINTER(i64)]
    L.gls_read_timing.restype = ctypes.c_int
    L.gls_get_dims.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.gls_get_dims.restype = ctypes.c_int
    cp = ctypes.c_char_p
    L.gls_solve_file.argtypes = [vp, cp, i64, i32, i64, cp, cp, i64, i64, i32, ctypes.POINTER(OocReport)]
    L.gls_solve_file.restype = ctypes.c_int
    L.gls_select_block_size.argtypes = [i64, i32, i32, i32, i64, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.POINTER(i32)]
    L.gls_select_block_size.restype = i64
    L.gls_set_stream_report.argtypes = [vp, i32]
    L.gls_set_stream_report.restype = ctypes.c_int
    L.gls_read_stream_report.argtypes = [vp, ctypes.POINTER(StreamReport)]
    L.gls_read_stream_report.restype = ctypes.c_int
    L.gls_gwfgls_create.argtypes = [i64, i32, i32, dp, dp, dp, ctypes.POINTER(vp)]
    L.gls_gwfgls_create.restype = ctypes.c_int
    L.gls_gwfgls_solve.argtypes = [vp, dp, i64, dp, dp, i32]
    L.gls_gwfgls_solve.restype = ctypes.c_int
    L.gls_gwfgls_launches.argtypes = [vp]
    L.gls_gwfgls_launches.restype = i64
    L.gls_gwfgls_destroy.argtypes = [vp]
    L.gls_gwfgls_destroy.restype = None
    L.gls_create_adopt_int8.argtypes = [i64, i32, i32, ctypes.POINTER(vp)]
    L.gls_create_adopt_int8.restype = ctypes.c_int
    L.gls_shared_view_ex.argtypes = [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.gls_shared_view_ex.restype = ctypes.c_int
    L.gls_dist_create.argtypes = [i64, i32, i32, i64, i32, i32, dp, dp, dp, ctypes.POINTER(vp)]
    L.gls_dist_create.restype = ctypes.c_int
    L.gls_dist_info.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.gls_dist_info.restype = ctypes.c_int
    L.gls_dist_buffer.argtypes = [vp, i32, i64, ctypes.POINTER(vp), ctypes.POINTER(i64)]
    L.gls_dist_buffer.restype = ctypes.c_int
    L.gls_dist_step.argtypes = [vp, i32, i64]
    L.gls_dist_step.restype = ctypes.c_int
    L.gls_dist_finish.argtypes = [vp, ctypes.POINTER(vp)]
    L.gls_dist_finish.restype = ctypes.c_int
    L.gls_dist_failed_pivot.argtypes = [vp]
    L.gls_dist_failed_pivot.restype = i64
    L.gls_dist_launches.argtypes = [vp]
    L.gls_dist_launches.restype = i64
    L.gls_dist_destroy.argtypes = [vp]
    L.gls_dist_destroy.restype = None
    L.gls_release_cached_memory.argtypes = []
    L.gls_release_cached_memory.restype = ctypes.c_int
    _lib = L
    return L


def load_gen():
    """libglsgen_dev.so: device genotype generator (test / bench input only)."""
    global _gen
    if _gen is None:
        path = _build.lib_path("libglsgen_dev.so")
        if not os.path.exists(path):
            _build.build()
        G = ctypes.CDLL(path)
        G.glsgen_dev_xr.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64,
                                    ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        G.glsgen_dev_xr.restype = ctypes.c_int
        _gen = G
    return _gen


def _ptr(a, dtype: str = "float64"):
    """Raw pointer of a torch tensor / numpy array (must be contiguous, right dtype); None -> NULL."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch
        assert a.is_contiguous(), "tensor must be contiguous"
        assert str(a.dtype).endswith(dtype), "expected %s, got %s" % (dtype, a.dtype)
        return a.data_ptr()
    import numpy as np
    assert isinstance(a, np.ndarray) and a.flags.c_contiguous and a.dtype == np.dtype(dtype)
    return a.ctypes.data


def select_block_size(n: int, p: int, pR: int, elem_bytes: int, mem_limit_bytes: int,
                      compute_groups_per_s: float, io_bytes_per_s: float, io_latency_s: float = 0.0):
    """gls_select_block_size (§4.3): (block problems, io_bound)."""
    flag = ctypes.c_int32()
    k = load().gls_select_block_size(n, p, pR, elem_bytes, mem_limit_bytes, compute_groups_per_s,
                                     io_bytes_per_s, io_latency_s, ctypes.byref(flag))
    return int(k), bool(flag.value)


def release_cached_memory() -> None:
    """gls_release_cached_memory: hand the pool memory cached by destroyed contexts back to the driver."""
    rc = load().gls_release_cached_memory()
    if rc:
        raise GLSError(rc, error_string(rc))


def device_bytes(ptr: int, nbytes: int):
    """A zero-copy torch uint8 CUDA tensor over `nbytes` of library-owned device memory at `ptr`."""
    import torch

    class _Raw:
        def __init__(self, p, nb):
            self.__cuda_array_interface__ = {"shape": (nb,), "typestr": "|u1",
                                             "data": (p, False), "version": 2, "strides": None}

    return torch.as_tensor(_Raw(ptr, nbytes), device="cuda")


def error_string(code: int) -> str:
    return load().gls_error_string(code).decode()


class Context:
    """gls_ctx wrapper.  Context(n, pL, pR, M, X_L, y) runs gls_create on the current device;
    async_create=True runs gls_create_async (M, X_L, y are kept referenced until the first
    synchronising call; a non-SPD M raises there)."""

    def __init__(self, n: int, pL: int, pR: int, M=None, X_L=None, y=None, adopt: bool = False,
                 int8_only: bool = False, _handle=None, async_create: bool = False):
        L = load()
        self._lib = L
        self.n, self.pL, self.pR, self.p = n, pL, pR, pL + pR
        self.int8_only = int8_only
        self.share_flags = 0
        h = ctypes.c_void_p()
        if _handle is not None:  # a context the library built elsewhere (gls_dist_finish)
            self._h = _handle
            self.failed_pivot = -1
            return
        if adopt and int8_only:
            rc = L.gls_create_adopt_int8(n, pL, pR, ctypes.byref(h))
        elif adopt:
            rc = L.gls_create_adopt(n, pL, pR, ctypes.byref(h))
        else:
            create = L.gls_create_async if async_create else L.gls_create
            rc = create(n, pL, pR, _ptr(M), _ptr(X_L) if pL > 0 else None, _ptr(y), ctypes.byref(h))
        self._h = h
        self.failed_pivot = -1
        self._borrowed = (M, X_L, y) if async_create else None  # read in stream order until synchronised
        if rc != GLS_OK:
            msg = error_string(rc)
            if h.value:
                self.failed_pivot = L.gls_failed_pivot(h)
                msg += " -- " + L.gls_last_error(h).decode()
                L.gls_destroy(h)
                self._h = ctypes.c_void_p()
            raise GLSError(rc, msg)

    # -- helpers
    def _check(self, rc: int):
        if rc != GLS_OK:
            if rc == GLS_ERR_NOT_SPD:  # an asynchronous create's factorisation failed
                self.failed_pivot = self._lib.gls_failed_pivot(self._h)
            raise GLSError(rc, error_string(rc) + " -- " + self._lib.gls_last_error(self._h).decode())

    def solve_block(self, X_R, m_blk: int, b_out, status_out=None, async_: bool = False):
        self._check(self._lib.gls_solve_block_ex(self._h, _ptr(X_R), m_blk, _ptr(b_out),
                                                 _ptr(status_out, "int32"), 1 if async_ else 0))

    def solve_block_i8(self, G, m_blk: int, b_out, status_out=None, async_: bool = False, ldg: int | None = None):
        """X_R as int8 genotype codes: G of shape (m_blk*pR, ldg) (row j = column j of X_R)."""
        ld = ldg if ldg is not None else int(G.shape[-1])
        self._check(self._lib.gls_solve_block_i8(self._h, _ptr(G, "int8"), ld, m_blk, _ptr(b_out),
                                                 _ptr(status_out, "int32"), 1 if async_ else 0))

    def solve_file(self, xr_path: str, m: int, b_path: str, status_path: str | None = None, elem_bytes: int = 8,
                   xr_offset: int = 0, block_groups: int = 65536, warmup_groups: int = 0,
                   mode: int = GLS_OOC_ASYNC) -> dict:
        """Out-of-core solve from a file (gls_solve_file; Alg. 7 when mode=GLS_OOC_SYNC, Alg. 8 when
        GLS_OOC_ASYNC).  Returns the overlap report as a dict."""
        rep = OocReport()
        enc = lambda x: x.encode() if x is not None else None
        self._check(self._lib.gls_solve_file(self._h, enc(xr_path), xr_offset, elem_bytes, m, enc(b_path),
                                             enc(status_path), block_groups, warmup_groups, mode,
                                             ctypes.byref(rep)))
        return rep.as_dict()

    def set_timing(self, enable: bool = True):
        self._check(self._lib.gls_set_timing(self._h, 1 if enable else 0))

    def read_timing(self):
        """{'int8_ms', 'fp64_ms', 'conv_ms', 'launches'} summed since the last read (synchronises)."""
        a, b, c, k = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        self._check(self._lib.gls_read_timing(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                              ctypes.byref(k)))
        return {"int8_ms": a.value, "fp64_ms": b.value, "conv_ms": c.value, "launches": k.value}

    def set_stream_report(self, enable: bool = True):
        self._check(self._lib.gls_set_stream_report(self._h, 1 if enable else 0))

    def read_stream_report(self):
        """Overlap accounting of the host chunks streamed since the last read (synchronises)."""
        r = StreamReport()
        self._check(self._lib.gls_read_stream_report(self._h, ctypes.byref(r)))
        return r.as_dict()

    def sync(self):
        self._check(self._lib.gls_sync(self._h))

    def set_stream(self, stream_handle: int | None):
        self._check(self._lib.gls_set_stream(self._h, stream_handle))

    def set_block_cols(self, cols: int):
        self._check(self._lib.gls_set_block_cols(self._h, cols))

    def shared_view(self, flags: int | None = None):
        """gls_shared_view_ex with `flags` (default: self.share_flags; GLS_SHARE_INT8_ONLY lists only the
        int8 path's state -- what an int8-only receiver needs)."""
        ptrs = (ctypes.c_void_p * 8)()
        nbytes = (ctypes.c_int64 * 8)()
        cnt = ctypes.c_int32()
        f = self.share_flags if flags is None else flags
        self._check(self._lib.gls_shared_view_ex(self._h, f, ptrs, nbytes, ctypes.byref(cnt)))
        return [(ptrs[k], nbytes[k]) for k in range(cnt.value)]

    def shared_tensors(self, flags: int | None = None):
        """The shared-state buffers as zero-copy torch uint8 CUDA tensors (for dist.broadcast)."""
        return [device_bytes(p, nb) for p, nb in self.shared_view(flags)]

    def commit_shared(self):
        self._check(self._lib.gls_commit_shared(self._h))

    def set_path(self, path: int):
        """GLS_PATH_AUTO (int8 tensor cores for integer genotype blocks) or GLS_PATH_FP64."""
        self._check(self._lib.gls_set_path(self._h, path))

    def path_counts(self):
        """(int8 hot-kernel launches that did work, FP64 ones) -- synchronises the context."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._lib.gls_path_counts(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.gls_kernel_launches(self._h))

    def close(self):
        if self._h and self._h.value:
            self._lib.gls_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def gen_xr_device(seed: int, n: int, col0: int, ncols: int, X, ld: int | None = None, stream: int = 0):
    """Fill a CUDA float64 tensor X (shape (ncols, ld)) with genotype columns [col0, col0+ncols)."""
    rc = load_gen().glsgen_dev_xr(seed, n, col0, ncols, X.data_ptr(), ld or n, stream)
    if rc != 0:
        raise GLSError(GLS_ERR_CUDA, "glsgen_dev_xr failed with cudaError %d" % rc)


class Gwfgls:
    """GenABEL's gwfgls (Alg. 6) on the B200 kernels (gls_gwfgls_*): a ladder rung for
    Table II's cost comparison.  Device tensors only for solve()."""

    def __init__(self, n: int, pL: int, pR: int, M, X_L, y):
        L = load()
        self._lib = L
        self.n, self.pL, self.pR, self.p = n, pL, pR, pL + pR
        h = ctypes.c_void_p()
        rc = L.gls_gwfgls_create(n, pL, pR, _ptr(M), _ptr(X_L) if pL > 0 else None, _ptr(y), ctypes.byref(h))
        if rc != GLS_OK:
            raise GLSError(rc, error_string(rc))
        self._h = h

    def solve(self, X_R, m_blk: int, b_out, status_out=None, mode: int = GLS_GWFGLS_GEMV):
        rc = self._lib.gls_gwfgls_solve(self._h, _ptr(X_R), m_blk, _ptr(b_out), _ptr(status_out, "int32"), mode)
        if rc != GLS_OK:
            raise GLSError(rc, error_string(rc))

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.gls_gwfgls_launches(self._h))

    def close(self):
        if self._h and self._h.value:
            self._lib.gls_gwfgls_destroy(self._h)
        self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistFactor:
    """gls_dist_* (include/gls.h): this rank's share of the distributed create of an M beyond one GPU
    (NEXT-3).  multi.dist_create runs the protocol; this class only marshals."""

    def __init__(self, n: int, pL: int, pR: int, nb: int, nranks: int, rank: int, M, X_L, y):
        L = load()
        self._lib = L
        self.n, self.pL, self.pR = n, pL, pR
        self.nranks, self.rank = nranks, rank
        h = ctypes.c_void_p()
        rc = L.gls_dist_create(n, pL, pR, nb, nranks, rank, _ptr(M), _ptr(X_L) if pL > 0 else None, _ptr(y),
                               ctypes.byref(h))
        if rc != GLS_OK:
            raise GLSError(rc, error_string(rc))
        self._h = h
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        L.gls_dist_info(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
        self.nb, self.nblocks, self.nloc = a.value, b.value, c.value

    def buffer(self, which: int, k: int = 0):
        """Zero-copy uint8 CUDA tensor over a gls_dist buffer (GLS_DIST_*)."""
        p, nb = ctypes.c_void_p(), ctypes.c_int64()
        rc = self._lib.gls_dist_buffer(self._h, which, k, ctypes.byref(p), ctypes.byref(nb))
        if rc != GLS_OK:
            raise GLSError(rc, error_string(rc))
        return device_bytes(p.value, nb.value)

    def step(self, phase: int, k: int = 0) -> int:
        """gls_dist_step; returns the return code (GLS_ERR_NOT_SPD is reported, not raised)."""
        rc = self._lib.gls_dist_step(self._h, phase, k)
        if rc not in (GLS_OK, GLS_ERR_NOT_SPD):
            raise GLSError(rc, error_string(rc))
        return rc

    @property
    def failed_pivot(self) -> int:
        return int(self._lib.gls_dist_failed_pivot(self._h))

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.gls_dist_launches(self._h))

    def finish(self) -> Context:
        h = ctypes.c_void_p()
        rc = self._lib.gls_dist_finish(self._h, ctypes.byref(h))
        if rc != GLS_OK:
            raise GLSError(rc, error_string(rc))
        ctx = Context(self.n, self.pL, self.pR, int8_only=True, _handle=h)
        ctx.share_flags = GLS_SHARE_INT8_ONLY
        return ctx

    def close(self):
        if self._h and self._h.value:
            self._lib.gls_dist_destroy(self._h)
        self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
