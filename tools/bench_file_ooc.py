#!/usr/bin/env python
"""Out-of-core from secondary storage (NEXT-1 of SURVEY §8(f); §4, Alg. 7 vs Alg. 8).

Writes a config-4-shaped X_R stream (n = 1e4, pL = 3, pR = 1; genotype codes int8 or FP64) to a file,
evicts it from the page cache (fsync + POSIX_FADV_DONTNEED), measures the raw sequential read rate of
the file, then times gls_solve_file in the synchronous mode (Alg. 7) and the double-buffered mode
(Alg. 8) -- each from a cold page cache -- and prints one JSON line with both, the overlap reports
and the roofline max(t_read, t_compute).  Results are checked bitwise between the two modes.

    python tools/bench_file_ooc.py [--m 1000000] [--elem 1|8] [--block 151552] [--warmup 18944] [--dir /tmp]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1210_7325_b200 as pkg  # noqa: E402


def evict(path):
    fd = os.open(path, os.O_RDONLY)
    os.fsync(fd)
    os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
    os.close(fd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1_000_000)
    ap.add_argument("--elem", type=int, default=1, choices=[1, 8])
    ap.add_argument("--block", type=int, default=0, help="SNPs per block (default 4 waves of tiles for int8 "
                    "codes, 1 wave for FP64: two pinned workspaces of this size are allocated)")
    ap.add_argument("--warmup", type=int, default=148 * 128)
    ap.add_argument("--dir", default="/tmp")
    args = ap.parse_args()
    if args.block <= 0:
        args.block = 148 * 128 * (4 if args.elem == 1 else 1)
    cfg = gen.CONFIGS[4]
    n, pL, pR, m = cfg.n, cfg.pL, cfg.pR, args.m
    P = gen.config_problem(cfg)
    xr = os.path.join(args.dir, "gls_xr_%d.bin" % args.elem)
    bf = os.path.join(args.dir, "gls_b.bin")
    # generate the stream blockwise on the GPU, write it to the file (untimed)
    chunk = 65536
    tmp = torch.empty((chunk, n), dtype=torch.float64, device="cuda")
    with open(xr, "wb") as f:
        for c in range(0, m * pR, chunk):
            k = min(chunk, m * pR - c)
            pkg.gen_xr_device(gen.DEFAULT_SEED, n, c, k, tmp[:k])
            blk = tmp[:k].to(torch.int8) if args.elem == 1 else tmp[:k]
            f.write(blk.cpu().numpy().tobytes())
    del tmp
    size = os.path.getsize(xr)
    # raw sequential read rate of this file from a cold cache, read the way the engine reads it
    # (O_DIRECT, 64 MiB requests into a page-aligned buffer): the I/O roofline
    import mmap
    evict(xr)
    buf = mmap.mmap(-1, 64 << 20)
    t0 = time.perf_counter()
    fd = os.open(xr, os.O_RDONLY | getattr(os, "O_DIRECT", 0))
    off = 0
    while True:
        got = os.preadv(fd, [buf], off)
        if got <= 0:
            break
        off += got
    os.close(fd)
    t_read = time.perf_counter() - t0
    read_gbs = size / t_read / 1e9
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out = {}
    bits = {}
    for name, mode in (("sync_alg7", pkg.GLS_OOC_SYNC), ("async_alg8", pkg.GLS_OOC_ASYNC)):
        evict(xr)
        t0 = time.perf_counter()
        with pkg.Context(n, pL, pR, d(P.M), d(P.XL), d(P.y)) as ctx:
            rep = ctx.solve_file(xr, m, bf, elem_bytes=args.elem, block_groups=args.block,
                                 warmup_groups=args.warmup, mode=mode)
        dt = time.perf_counter() - t0
        bits[name] = np.fromfile(bf)
        rep["snps_per_s"] = m / rep["wall_s"]  # the engine's wall time (create and pinning excluded)
        rep["with_create_and_pinning_s"] = dt
        out[name] = rep
    same = bool(np.array_equal(bits["sync_alg7"], bits["async_alg8"]))
    # compute-only rate of the same blocks from pinned host memory is the in-core e2e; here the
    # compute share is what the async mode can hide
    t_comp = out["async_alg8"]["compute_s"]
    roof = max(t_read, t_comp)
    line = {"metric": "GLS solves (SNPs)/sec, out-of-core from secondary storage (Alg. 7 vs Alg. 8)",
            "value": out["async_alg8"]["snps_per_s"], "unit": "SNPs/s", "n_gpus": 1,
            "config": {"workload": "config4 shape from a file: n=%d pL=%d pR=%d, m=%d, X_R as %s (%.1f GB)"
                                   % (n, pL, pR, m, "int8 codes" if args.elem == 1 else "FP64", size / 1e9),
                       "block_snps": args.block, "warmup_block_snps": args.warmup, "file": xr},
            "raw_read": {"seconds": t_read, "GBps": read_gbs, "method": "O_DIRECT, 64 MiB requests, cold"},
            "roofline": {"bound": "disk" if t_read >= t_comp else "compute", "t_read_s": t_read,
                         "t_compute_s": t_comp, "frac": roof / out["async_alg8"]["wall_s"]},
            "sync_over_async": out["sync_alg7"]["wall_s"] / out["async_alg8"]["wall_s"],
            "modes": out, "bitwise_equal_sync_async": same}
    print(json.dumps(line))
    os.remove(xr)
    os.remove(bf)


if __name__ == "__main__":
    main()
