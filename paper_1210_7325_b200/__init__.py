"""B200-native hot path of HP-GWAS / OOC-HP-GWAS (arXiv 1210.7325).

`gls` is the ctypes binding of libgls.so (C ABI in include/gls.h); `build` compiles the
in-tree CUDA libraries for sm_100a.  See DESIGN.md.
"""
from .gls import (GLS_GWFGLS_GEMM, GLS_GWFGLS_GEMV, GLS_OOC_ASYNC, GLS_OOC_SYNC, GLS_PATH_AUTO,  # noqa: F401
                  GLS_PATH_FP64, Context, GLSError, Gwfgls, gen_xr_device, load, release_cached_memory,
                  select_block_size)
