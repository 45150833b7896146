"""Run one (n, pL, pR, m) case through the C ABI in this process and compare with the oracle.
usage: python tools/bisect_case.py n pL pR m [host]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import gen, oracle
import paper_1210_7325_b200 as pkg
from _util import guarded_rel_err
n, pL, pR, m = map(int, sys.argv[1:5])
P = gen.make_problem(n, pL, pR, with_sex=pL >= 2, seed=7)
XR = gen.make_XR(7, n, 0, m * pR)
b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
with pkg.Context(n, pL, pR, d(P.M), d(P.XL) if pL else None, d(P.y)) as ctx:
    b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
    st = torch.empty(m, dtype=torch.int32, device="cuda")
    ctx.solve_block(XR if len(sys.argv) > 5 else d(XR), m, b, st)
print("case", sys.argv[1:], "err %.3e" % guarded_rel_err(b.cpu().numpy(), b_or), "status_ok", bool((st.cpu().numpy() == st_or).all()))
