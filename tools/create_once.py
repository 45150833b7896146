"""One gls_create at n (diagnostics for ncu launch lists): python tools/create_once.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
P = gen.make_problem(n, 3, 1)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
for _ in range(2):
    with pkg.Context(n, 3, 1, d(P.M), d(P.XL), d(P.y)) as c:
        torch.cuda.synchronize()
