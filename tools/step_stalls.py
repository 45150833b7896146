"""Diagnostics: where the occasional 55-93 ms outlier steps of the config-2 bench loop come from.
Runs bench.py's step (gls_create + gls_solve_block on 1e6 SNPs in HBM + close) K times with host
timestamps around every call and CUDA events on the compute stream; with GLS_TRACE=1 the library
also prints the create's host-side phases.  usage: python tools/step_stalls.py [steps] [m]"""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg
import paper_1210_7325_b200.gls as g

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
cfg = gen.CONFIGS[2]
n, pL, pR = cfg.n, cfg.pL, cfg.pR
P = gen.config_problem(cfg)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
Md, XLd, yd = d(P.M), d(P.XL), d(P.y)
X = torch.empty((m * pR, n), dtype=torch.float64, device="cuda")
for c in range(0, m * pR, 65536):
    k = min(65536, m * pR - c)
    g.gen_xr_device(gen.DEFAULT_SEED, n, c, k, X[c:c + k])
b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
st = torch.empty(m, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
gc.collect()
gc.disable()

rows = []
for it in range(steps + 3):
    t = [time.perf_counter()]
    ctx = pkg.Context(n, pL, pR, Md, XLd, yd)
    t.append(time.perf_counter())                     # 1: create returned
    ctx.set_stream(stream.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.solve_block(X, m, b, st, async_=True)
    e1.record(stream)
    t.append(time.perf_counter())                     # 2: solve enqueued
    ctx.sync()
    t.append(time.perf_counter())                     # 3: solve done
    ctx.close()
    t.append(time.perf_counter())                     # 4: closed
    ms = [1e3 * (t[i + 1] - t[i]) for i in range(4)]
    rows.append((it, ms, e0.elapsed_time(e1)))
    print("step %2d  create %7.2f  enqueue %6.2f  sync %7.2f  close %6.2f  | solve(ev) %7.2f  total %7.2f"
          % (it, ms[0], ms[1], ms[2], ms[3], rows[-1][2], 1e3 * (t[4] - t[0])), flush=True)
