"""Time gls_create (potrf + inverse + shared transforms) at several n; prints ms per create."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg
for n in [int(a) for a in sys.argv[1:]] or [1500, 10000]:
    P = gen.make_problem(n, 3, 1)
    Md, XLd, yd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (P.M, P.XL, P.y))
    ts = []
    for r in range(5):
        torch.cuda.synchronize(); t = time.perf_counter()
        c = pkg.Context(n, 3, 1, Md, XLd, yd)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
        L = c.kernel_launches
        c.close()
    print("create n=%d: %.2f ms (min of 5; %d launches)" % (n, 1e3 * min(ts[1:]), L))
