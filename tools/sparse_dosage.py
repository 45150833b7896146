"""Mixed genotype / dosage blocks (diagnostics for the per-problem path choice, reading A16):
config-2 shape (n = 1e4, p = 4), m SNPs in HBM of which a fraction hold one non-integer value; solve time
and path launches for fractions 0, 0.1 %, 1 %, 10 %, 100 %, and the all-FP64 path for comparison.
usage: python tools/sparse_dosage.py [m]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg

m = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
cfg = gen.CONFIGS[2]
n, pL, pR = cfg.n, cfg.pL, cfg.pR
P = gen.config_problem(cfg)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
Md, XLd, yd = d(P.M), d(P.XL), d(P.y)
X0 = torch.empty((m * pR, n), dtype=torch.float64, device="cuda")
for c in range(0, m * pR, 65536):
    k = min(65536, m * pR - c)
    pkg.gen_xr_device(gen.DEFAULT_SEED, n, c, k, X0[c:c + k])
b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
rng = np.random.default_rng(5)
with pkg.Context(n, pL, pR, Md, XLd, yd) as ctx:
    for frac, path in ((0.0, None), (0.001, None), (0.01, None), (0.1, None), (1.0, None), (0.0, "fp64")):
        X = X0.clone() if frac else X0
        nb = int(round(frac * m))
        if nb:
            rows = torch.from_numpy(np.sort(rng.choice(m * pR, nb, replace=False))).cuda()
            X[rows, 17] += 0.5
        ctx.set_path(pkg.GLS_PATH_FP64 if path else pkg.GLS_PATH_AUTO)
        a0 = ctx.path_counts()
        ts = []
        for rep in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            ctx.solve_block(X, m, b)
            torch.cuda.synchronize()
            ts.append(1e3 * (time.perf_counter() - t))
        a1 = ctx.path_counts()
        print("dosage fraction %-6g %-5s solve %8.1f ms  (%.3g SNPs/s)  int8 / FP64 launches %d / %d"
              % (frac, path or "auto", min(ts), m / (min(ts) / 1e3), a1[0] - a0[0], a1[1] - a0[1]), flush=True)
        del X
