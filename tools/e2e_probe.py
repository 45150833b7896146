"""Breakdown of one e2e step (host buffers through the C ABI): create, solve_block_i8 (or, with a
third argument "f64", solve_block on FP64 host X_R), close.
usage: python tools/e2e_probe.py [config] [reps] [i8|f64] [m]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg

pkg.load()
cfg = gen.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
mode = sys.argv[3] if len(sys.argv) > 3 else "i8"
n, pL, pR, m = cfg.n, cfg.pL, cfg.pR, cfg.m
if len(sys.argv) > 4:
    m = int(sys.argv[4])
m -= m % 64
P = gen.config_problem(cfg)
Mh = torch.from_numpy(P.M).pin_memory()
XLh = torch.from_numpy(np.ascontiguousarray(P.XL)).pin_memory()
yh = torch.from_numpy(P.y).pin_memory()
Xd = torch.empty((m * pR, n), dtype=torch.float64, device="cuda")
pkg.gen_xr_device(gen.DEFAULT_SEED, n, 0, m * pR, Xd)
Gh = Xd.to(torch.int8).cpu().pin_memory() if mode == "i8" else Xd.cpu().pin_memory()
del Xd
bh = torch.empty((m, pL + pR), dtype=torch.float64, pin_memory=True)
sh = torch.empty(m, dtype=torch.int32, pin_memory=True)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = pkg.Context(n, pL, pR, Mh, XLh, yh)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if mode == "i8":
        ctx.solve_block_i8(Gh, m, bh, sh)
    else:
        ctx.solve_block(Gh, m, bh, sh)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ctx.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print("rep %d: create %.2f ms  solve %.2f ms  close %.2f ms  total %.2f ms -> %.3g SNPs/s"
          % (r, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t3 - t0), m / (t3 - t0)), flush=True)
