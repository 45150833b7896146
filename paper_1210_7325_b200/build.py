"""Build the in-tree native libraries with nvcc for sm_100a.

    libgls.so         -- the product: C ABI of include/gls.h (csrc/gls_api.cu, dgemm.cu,
                         chol_inv.cu, fused_trsm_gls.cu)
    libglsgen_dev.so  -- device-side synthetic genotype generator (csrc/gen_device.cu),
                         used by tests and bench.py to fill X_R in HBM

No PyTorch types cross the boundary; torch is only used by callers for device memory,
streams and process groups.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-Xcompiler", "-Wall"]

LIBS = {
    "libgls.so": ["gls_api.cu", "dgemm.cu", "chol_inv.cu", "fused_trsm_gls.cu", "ozaki_gls.cu", "ooc_file.cu",
                  "gwfgls.cu", "dist_create.cu"],
    "libglsgen_dev.so": ["gen_device.cu"],
}
DEPS = ["gls_internal.cuh", "umma.cuh", os.path.join("..", "..", "include", "gls.h")]


def lib_path(name: str) -> str:
    return os.path.join(PKG, name)


def _stale(out: str, srcs) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False) -> None:
    for name, files in LIBS.items():
        srcs = [os.path.join(CSRC, f) for f in files]
        deps = srcs + [os.path.normpath(os.path.join(CSRC, d)) for d in DEPS]
        out = lib_path(name)
        if not force and not _stale(out, deps):
            continue
        tmp = out + ".tmp%d" % os.getpid()
        cmd = [NVCC] + ARCH + FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", tmp] + srcs
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(tmp, out)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
