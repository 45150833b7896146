"""Diagnostics: per-buffer digests of the shared state gls_create builds (T digits, packed T, aux, ...)
at the given n -- run twice under different scheduling switches (GLS_DGEMM_SCHED, GLS_SPLIT_FRAC, ...)
to show a change is bitwise neutral.  usage: python tools/create_digest.py n [n ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg
from paper_1210_7325_b200 import multi

for n in [int(a) for a in sys.argv[1:]] or [1500, 10000]:
    P = gen.make_problem(n, 3, 1)
    Md, XLd, yd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (P.M, P.XL, P.y))
    with pkg.Context(n, 3, 1, Md, XLd, yd) as c:
        print("n=%d digest %s" % (n, " ".join("%016x" % (d & (2**64 - 1)) for d in multi.shared_state_digest(c))))
