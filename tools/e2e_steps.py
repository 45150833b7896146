"""bench.py's e2e step (gls_create_async from pinned host M, stream report on, gls_solve_block_i8 of
pinned host codes, read_stream_report, close) K times with host timestamps around every call.
usage: python tools/e2e_steps.py [config] [steps]   (GLS_RES_CACHE=0 for the uncached A/B)"""
import gc, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg

pkg.load()
cfg = gen.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n, pL, pR, m = cfg.n, cfg.pL, cfg.pR, cfg.m
P = gen.config_problem(cfg)
Mh = torch.from_numpy(P.M).pin_memory()
XLh = torch.from_numpy(np.ascontiguousarray(P.XL)).pin_memory()
yh = torch.from_numpy(P.y).pin_memory()
Xd = torch.empty((m * pR, n), dtype=torch.float64, device="cuda")
pkg.gen_xr_device(gen.DEFAULT_SEED, n, 0, m * pR, Xd)
Gh = Xd.to(torch.int8).cpu().pin_memory()
del Xd
bh = torch.empty((m, pL + pR), dtype=torch.float64, pin_memory=True)
sh = torch.empty(m, dtype=torch.int32, pin_memory=True)
gc.collect()
gc.disable()
for r in range(steps + 1):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    ctx = pkg.Context(n, pL, pR, Mh, XLh, yh, async_create=True)
    t.append(time.perf_counter())
    ctx.set_stream_report(True)
    ctx.solve_block_i8(Gh, m, bh, sh)
    t.append(time.perf_counter())
    rep = ctx.read_stream_report()
    t.append(time.perf_counter())
    ctx.close()
    t.append(time.perf_counter())
    ms = [1e3 * (t[i + 1] - t[i]) for i in range(4)]
    print("step %2d: create_async %.2f  solve %.2f  report %.2f  close %.2f  total %.2f ms (stream wall %.2f)"
          % (r, *ms, 1e3 * (t[4] - t[0]), rep["wall_ms"]), flush=True)
