"""Diagnostics: why gls_create is slower inside the bench step (right after an int8 solve) than
standalone.  Config 2 (n = 1e4, 1e6 SNPs in HBM); per mode, 3 x [create, solve] and the create of
the next round is timed after: nothing (the bench order), a 0.5 s sleep (power/clock recovery), or a
512 MiB fill (L2 refilled with normal-priority lines).  Set GLS_OZ_UNPIN=1 to A/B the V-step
evict_first loads.  usage: python tools/create_after_solve.py [m]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg
import paper_1210_7325_b200.gls as g

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
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
junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def create():
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx = pkg.Context(n, pL, pR, Md, XLd, yd)
    torch.cuda.synchronize()
    return ctx, 1e3 * (time.perf_counter() - t)


def solve(ctx):
    ctx.set_timing(True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx.solve_block(X, m, b)
    torch.cuda.synchronize()
    tm = ctx.read_timing()
    return 1e3 * (time.perf_counter() - t), tm


for mode in ["none", "sleep", "fill", "none"]:
    cr, sv, k8 = [], [], []
    ctx, _ = create()
    for rep in range(3):
        s, tm = solve(ctx)
        ctx.close()
        if mode == "sleep":
            time.sleep(0.5)
        elif mode == "fill":
            junk.fill_(rep + 1)
        ctx, c = create()
        cr.append(c)
        sv.append(s)
        k8.append(tm["int8_ms"])
    ctx.close()
    print("unpin=%s after=%-5s create %s ms | solve %s ms | int8 kernel %s ms" % (
        os.environ.get("GLS_OZ_UNPIN", "0"), mode, " ".join("%.1f" % v for v in cr),
        " ".join("%.1f" % v for v in sv), " ".join("%.1f" % v for v in k8)), flush=True)
