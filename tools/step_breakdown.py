"""Host-side breakdown of bench.py's config-2 step (diagnostics): gls_create, the solve, the sync, the
destroy, with perf_counter stamps (every phase ends in a device sync).  usage: step_breakdown.py [m]
[timing] [smi]: timing = per-launch CUDA events + read_timing as bench.py does; smi = an nvidia-smi
-lms 200 sampler running meanwhile (bench.py's clock sampler)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg
cfg = gen.CONFIGS[2]
n, pL, pR, m = cfg.n, cfg.pL, cfg.pR, int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
P = gen.config_problem(cfg)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
Md, XLd, yd = d(P.M), d(P.XL), d(P.y)
X = torch.empty((m * pR, n), dtype=torch.float64, device="cuda")
for c in range(0, m * pR, 65536):
    k = min(65536, m * pR - c)
    pkg.gen_xr_device(gen.DEFAULT_SEED, n, c, k, X[c:c + k])
b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
st = torch.empty(m, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
opts = sys.argv[2:]
if "smi" in opts:
    import subprocess
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader",
                            "-lms", "200"], stdout=subprocess.DEVNULL)
for rep in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ctx = pkg.Context(n, pL, pR, Md, XLd, yd)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    ctx.set_stream(s.cuda_stream)
    if "timing" in opts:
        ctx.set_timing(True)
    ctx.solve_block(X, m, b, st, async_=True)
    t2 = time.perf_counter()
    ctx.sync()
    if "timing" in opts:
        ctx.read_timing()
        ctx.path_counts()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    ctx.close()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print("rep %d: create %.1f  solve-issue %.1f  solve-wait %.1f  destroy %.1f  total %.1f ms" %
          (rep, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3), 1e3 * (t4 - t0)), flush=True)
