"""Small cases of the hot path for compute-sanitizer (tools/sanitize.sh runs ONE tool per call).

Covers every kernel family of the path at the smallest sizes that reach it:
  * n = 1500, pL = 3, pR = 1: gls_create (recursive chol_inv: leaves, 128-row nodes, split-K and TMA
    DGEMMs), the int8 tcgen05 kernel with the standalone conversion pass, the FP64 DMMA kernel
    (GLS_PATH_FP64), and the host-streamed Alg. 8 path (pinned host X_R, 3 chunks);
  * n = 1500, pL = 16, pR = 4 (p = 20): the separate posv kernel of the int8 path;
  * n = 4096, pL = 3, pR = 1, two waves + a ragged tail: the convert-ahead warps of the int8 kernel.
Every result is compared with the oracle on a sample (the oracle is test infrastructure; this script
is a tool, like tests/).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import oracle
import paper_1210_7325_b200 as pkg

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from _util import guarded_rel_err  # noqa: E402


def case(n, pL, pR, m, sample, fp64=True, host=True):
    P = gen.make_problem(n, pL, pR, with_sex=True, seed=gen.DEFAULT_SEED)
    XR = gen.make_XR(gen.DEFAULT_SEED, n, 0, m * pR)
    sel = np.unique(np.concatenate([np.arange(min(sample, m)), [m - 1]]))
    cols = np.concatenate([np.arange(i * pR, (i + 1) * pR) for i in sel])
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, np.ascontiguousarray(XR[cols]), pR)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    p = pL + pR
    out = {}
    with pkg.Context(n, pL, pR, d(P.M), d(P.XL), d(P.y)) as ctx:
        Xd = d(XR)
        runs = [("auto", None, Xd)]
        if fp64:
            runs.append(("fp64", pkg.GLS_PATH_FP64, Xd))
        if host:
            runs.append(("host", None, torch.from_numpy(XR).pin_memory()))
        for name, path, X in runs:
            ctx.set_path(pkg.GLS_PATH_FP64 if path is not None else pkg.GLS_PATH_AUTO)
            if name == "host":
                ctx.set_block_cols(max(pR, (m // 3) * pR))
            b = torch.empty((m, p), dtype=torch.float64, device="cuda")
            st = torch.empty(m, dtype=torch.int32, device="cuda")
            ctx.solve_block(X, m, b, st)
            ctx.sync()
            bb, ss = b.cpu().numpy()[sel], st.cpu().numpy()[sel]
            assert np.array_equal(ss, st_or), name
            ok = st_or == 0
            err = guarded_rel_err(bb[ok], b_or[ok])
            assert err <= 1e-9, "%s: %.3e" % (name, err)
            out[name] = err
    print("n=%d pL=%d pR=%d m=%d: %s" % (n, pL, pR, m, " ".join("%s %.2e" % kv for kv in out.items())), flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    which = sys.argv[1:] or ["small", "p20", "ahead"]
    if "small" in which:
        case(1500, 3, 1, 3000, 64)
    if "p20" in which:
        case(1500, 16, 4, 600, 32, fp64=False, host=False)
    if "ahead" in which:
        case(4096, 3, 1, 2 * 148 * 128 + 77, 48, fp64=False, host=False)
    print("sanitize cases ok", flush=True)
