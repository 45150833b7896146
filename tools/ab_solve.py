"""A/B timing of the config-2 solve with a given libgls.so (diagnostics): only symbols every round-1
build exports.  usage: python tools/ab_solve.py LIB [m] [config] [i8]   (i8: X_R as int8 genotype codes
in HBM through gls_solve_block_i8 -- no conversion, no convert-ahead)"""
import ctypes, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gen
import paper_1210_7325_b200.gls as g

lib = ctypes.CDLL(sys.argv[1])
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
lib.gls_create.argtypes = [i64, i32, i32, vp, vp, vp, ctypes.POINTER(vp)]
lib.gls_solve_block_ex.argtypes = [vp, vp, i64, vp, vp, ctypes.c_int]
lib.gls_set_stream.argtypes = [vp, vp]
lib.gls_set_timing.argtypes = [vp, i32]
dpp = ctypes.POINTER(ctypes.c_double)
lib.gls_read_timing.argtypes = [vp, dpp, dpp, dpp, ctypes.POINTER(i64)]
lib.gls_destroy.argtypes = [vp]
cfg = gen.CONFIGS[int(sys.argv[3]) if len(sys.argv) > 3 else 2]
n = cfg.n
P = gen.config_problem(cfg)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
Md, XLd, yd = d(P.M), d(P.XL), d(P.y)
pL, pR = cfg.pL, cfg.pR
X = torch.empty((m * pR, n), dtype=torch.float64, device="cuda")
for c in range(0, m * pR, 65536):
    k = min(65536, m * pR - c)
    g.gen_xr_device(gen.DEFAULT_SEED, n, c, k, X[c:c + k])
b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
codes = len(sys.argv) > 4 and sys.argv[4] == "i8"
if codes:
    G = torch.empty((m * pR, n), dtype=torch.int8, device="cuda")
    for c in range(0, m * pR, 65536):
        G[c:c + 65536].copy_(X[c:c + 65536].to(torch.int8))
    del X
    lib.gls_solve_block_i8.argtypes = [vp, vp, i64, i64, vp, vp, ctypes.c_int]
s = torch.cuda.Stream()
for rep in range(4):
    h = vp()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    assert lib.gls_create(n, pL, pR, Md.data_ptr(), XLd.data_ptr(), yd.data_ptr(), ctypes.byref(h)) == 0
    t1 = time.perf_counter()
    lib.gls_set_stream(h, s.cuda_stream)
    lib.gls_set_timing(h, 1)
    if codes:
        assert lib.gls_solve_block_i8(h, G.data_ptr(), n, m, b.data_ptr(), None, 0) == 0
    else:
        assert lib.gls_solve_block_ex(h, X.data_ptr(), m, b.data_ptr(), None, 0) == 0
    t2 = time.perf_counter()
    a, bb, c, k = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    lib.gls_read_timing(h, ctypes.byref(a), ctypes.byref(bb), ctypes.byref(c), ctypes.byref(k))
    lib.gls_destroy(h)
    print("%s rep %d: create %.1f ms solve %.1f ms int8 kernel %.1f ms" % (os.path.basename(os.path.dirname(sys.argv[1])) or sys.argv[1], rep, 1e3 * (t1 - t0), 1e3 * (t2 - t1), a.value), flush=True)
