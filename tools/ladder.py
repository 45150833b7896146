#!/usr/bin/env python
"""The paper's algorithm ladder on B200 (NEXT-2 of SURVEY §8(f); Table II 338-421).

All three rungs run through the library's C ABI and its B200 kernels:
  black-box (Alg. 3): every problem solved alone -- a context (potrf + shared transforms) per problem,
                      with pL' = 0, pR' = p and X_R' = X_i = [X_L | X_Ri]           cost O(m n^3)
  seq-gls   (Alg. 4): one factorization; per problem all p columns of X_i whitened -- one context with
                      pL' = 0, pR' = p over the interleaved columns [X_L | X_Ri]    cost O(n^3 + m p n^2)
  hp-gwas   (Alg. 5): one factorization, X_L whitened once, per problem only X_Ri  cost O(n^3 + m n^2)
  gwfgls    (Alg. 6): GenABEL's listing on the library's gls_gwfgls_* kernels: explicit
                      M^{-1} = T^T T, W_L = M^{-1} X_L, per problem w = M^{-1} x_R as a gemv (listed) or
                      the block's gemvs as one GEMM ("gwfgls-gemm"), S_i = W^T X_i, gesv      cost O(n^3 + m n^2 + m n p^2)
Prints one JSON line with the measured problems/s of each rung, the ratios to hp-gwas next to
Table II's predictions (~n, ~p, 1, ~2), and the max deviation of each rung's b from hp-gwas's.
seq-gls and black-box take the FP64 tensor path (X_L holds a N(0,1) covariate, so their X_R' is not
integer); hp-gwas takes the int8 path (and, forced, the FP64 path: the same-arithmetic comparison).

    python tools/ladder.py [--n 1500] [--m 20000] [--m-blackbox 40]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1210_7325_b200 as pkg  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def interleave(XL, XR, pR):
    """X_R' for pL' = 0: problem i's columns = [X_L | X_Ri]  (rows of the (cols, n) arrays)."""
    m = XR.shape[0] // pR
    pL = XL.shape[0]
    out = np.empty((m * (pL + pR), XL.shape[1]))
    for i in range(m):
        out[i * (pL + pR):i * (pL + pR) + pL] = XL
        out[i * (pL + pR) + pL:(i + 1) * (pL + pR)] = XR[i * pR:(i + 1) * pR]
    return out


def timed_solve(n, pL, pR, M, XL, y, X, m, path=None):
    """Create a context (untimed), one warm-up solve, then the timed solve of m problems."""
    p = pL + pR
    with pkg.Context(n, pL, pR, M, XL, y) as ctx:
        if path is not None:
            ctx.set_path(path)
        b = torch.empty((m, p), dtype=torch.float64, device="cuda")
        ctx.solve_block(X, m, b)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.solve_block(X, m, b)
        torch.cuda.synchronize()
        return time.perf_counter() - t0, b.cpu().numpy()


def timed_gwfgls(n, pL, pR, M, XL, y, X, m, mode):
    """gwfgls (Alg. 6) on the device: create (untimed), a warm-up solve, then the timed solve."""
    with pkg.Gwfgls(n, pL, pR, M, XL, y) as g:
        b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
        g.solve(X, m, b, mode=mode)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.solve(X, m, b, mode=mode)
        torch.cuda.synchronize()
        return time.perf_counter() - t0, b.cpu().numpy()


def run(n, pL, pR, m, m_bb, seed=gen.DEFAULT_SEED, return_b=False, m_gemv=None):
    p = pL + pR
    P = gen.make_problem(n, pL, pR, with_sex=True, seed=seed)
    XR = gen.make_XR(seed, n, 0, m * pR)
    Md, XLd, yd = dev(P.M), dev(P.XL), dev(P.y)
    # hp-gwas (Alg. 5): the per-problem work is X_Ri only
    t_hp, b_hp = timed_solve(n, pL, pR, Md, XLd, yd, dev(XR), m)
    # the same on the FP64 path: Table II's algorithmic ratios at equal arithmetic
    t_hp64, _ = timed_solve(n, pL, pR, Md, XLd, yd, dev(XR), m, path=pkg.GLS_PATH_FP64)
    # seq-gls (Alg. 4): pL' = 0, pR' = p, X_i = [X_L | X_Ri] whitened whole for every problem
    t_sq, b_sq = timed_solve(n, 0, p, Md, None, yd, dev(interleave(P.XL, XR, pR)), m)
    # black-box (Alg. 3): a whole GLS solve, potrf included, per problem (first m_bb problems)
    Xs_h = interleave(P.XL, XR[:m_bb * pR], pR)
    b_bb = np.empty((m_bb, p))

    def bb(i):
        with pkg.Context(n, 0, p, Md, None, yd) as ctx:
            bi = torch.empty((1, p), dtype=torch.float64, device="cuda")
            ctx.solve_block(dev(Xs_h[i * p:(i + 1) * p]), 1, bi)
            b_bb[i] = bi.cpu().numpy()[0]

    bb(0)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(m_bb):
        bb(i)
    t_bb = time.perf_counter() - t0
    # gwfgls (Alg. 6): the listing's per-column gemv on the first m_gemv problems, and its BLAS-3 variant
    m_gv = min(m, m_gemv if m_gemv is not None else m)
    Xd = dev(XR)
    t_gv, b_gv = timed_gwfgls(n, pL, pR, Md, XLd, yd, Xd, m_gv, pkg.GLS_GWFGLS_GEMV)
    t_gm, b_gm = timed_gwfgls(n, pL, pR, Md, XLd, yd, Xd, m, pkg.GLS_GWFGLS_GEMM)
    rate = {"black-box": m_bb / t_bb, "seq-gls": m / t_sq, "hp-gwas": m / t_hp, "hp-gwas-fp64": m / t_hp64,
            "gwfgls": m_gv / t_gv, "gwfgls-gemm": m / t_gm}
    dev_rel = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
    out = {"n": n, "pL": pL, "pR": pR, "p": p, "m": m, "m_blackbox": m_bb,
            "problems_per_s": rate,
            "ratio_to_hp_gwas": {k: rate["hp-gwas"] / v for k, v in rate.items()},
            "ratio_to_hp_gwas_fp64_same_arithmetic": {k: rate["hp-gwas-fp64"] / rate[k]
                                                      for k in ("black-box", "seq-gls", "hp-gwas-fp64", "gwfgls",
                                                                "gwfgls-gemm")},
            "table2_prediction": {"black-box": "~n (= %d)" % n, "seq-gls": "~p (= %d)" % p, "hp-gwas": "1",
                                  "gwfgls": "~2 (flops; the listing's per-column gemv is memory-bound on top)"},
            "m_gwfgls_gemv": m_gv,
            "paths": {"hp-gwas": "int8 digit split (X_R integer)", "hp-gwas-fp64": "FP64 DMMA (forced)",
                      "seq-gls": "FP64 DMMA (X_R' holds the real covariates of X_L)",
                      "black-box": "FP64 DMMA + a factorization per problem",
                      "gwfgls": "FP64: explicit M^-1 (DMMA GEMM), one memory-bound gemv per column",
                      "gwfgls-gemm": "FP64: explicit M^-1, the block's gemvs as one DMMA GEMM"},
            "max_rel_dev_from_hp_gwas": {"seq-gls": dev_rel(b_sq, b_hp), "black-box": dev_rel(b_bb, b_hp[:m_bb]),
                                         "gwfgls": dev_rel(b_gv, b_hp[:m_gv]), "gwfgls-gemm": dev_rel(b_gm, b_hp)},
            "note": "solve time per rung after a warm-up (the m -> infinity cost of Table II); black-box "
                    "includes its per-problem factorization and runs on the first m_blackbox problems"}
    if return_b:
        out["_b"] = {"hp-gwas": b_hp, "seq-gls": b_sq, "black-box": b_bb, "gwfgls": b_gv, "gwfgls-gemm": b_gm}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1500)
    ap.add_argument("--m", type=int, default=200000)
    ap.add_argument("--m-blackbox", type=int, default=40)
    ap.add_argument("--m-gemv", type=int, default=2000, help="problems for gwfgls's per-column gemv rung")
    args = ap.parse_args()
    pkg.load()
    print(json.dumps({"metric": "algorithm ladder on B200 (Table II)",
                      **run(args.n, 3, 1, args.m, args.m_blackbox, m_gemv=args.m_gemv)}))


if __name__ == "__main__":
    main()
