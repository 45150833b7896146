"""NEXT-3 on the GPU: the distributed create (include/gls.h gls_dist_*, multi.dist_create) through the real
library, checked against the CPU oracle.

* world 1 (one process): the blocked right-looking factorisation with panel steps alone;
* world 2 (two processes on the one GPU over gloo -- NCCL refuses two ranks on one device; the ranks'
  kernels never wait on each other, the host moves the panels): each rank holds half of the column
  blocks of M and T, the resulting int8-only contexts carry bit-identical shared state, each solves its
  strong-scaling shard, and b matches the oracle;
* a non-SPD M stops every rank with the oracle's pivot; int8-only contexts refuse the FP64 path and
  non-integer X_R."""
import os

import numpy as np
import pytest

import gen
import oracle

from _util import assert_parity, record_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 71


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1210_7325_b200 as p
    p.load()
    return p


@pytest.mark.parametrize("n,pL,pR,nb,m", [(1000, 3, 1, 128, 300), (777, 16, 4, 256, 60), (300, 0, 2, 128, 90)])
def test_dist_create_world1_matches_oracle(pkg, n, pL, pR, nb, m):
    from paper_1210_7325_b200 import multi
    P = gen.make_problem(n, pL, pR, with_sex=pL >= 3, seed=SEED + n)
    XR = gen.make_XR(SEED + n, n, 0, m * pR)
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
    ctx = multi.dist_create(n, pL, pR, dev(P.M), dev(P.XL) if pL else None, dev(P.y), nb=nb)
    with ctx:
        b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
        st = torch.empty(m, dtype=torch.int32, device="cuda")
        ctx.solve_block(dev(XR), m, b, st)                     # integer doubles: converted, int8 path
        assert_parity(b.cpu().numpy(), st.cpu().numpy(), b_or, st_or, label="dist world 1")
        record_parity("dist create world 1, n=%d p=%d nb=%d" % (n, pL + pR, nb), b.cpu().numpy(), b_or, st_or)
        G = torch.from_numpy(XR.astype(np.int8)).cuda()
        b8 = torch.empty_like(b)
        ctx.solve_block_i8(G, m, b8)                          # genotype codes
        assert torch.equal(b8, b)
        with pytest.raises(pkg.GLSError) as e:
            ctx.set_path(pkg.GLS_PATH_FP64)
        assert e.value.code == 6
        XR2 = XR.copy()
        XR2[1, 2] = 0.5
        with pytest.raises(pkg.GLSError) as e:
            ctx.solve_block(dev(XR2), m, b)
        assert e.value.code == 1


def _rank_main(rank, world, init_file, out_dir, n, nb, m, bad):
    import torch
    import torch.distributed as dist

    import paper_1210_7325_b200 as p
    from paper_1210_7325_b200 import multi

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method="file://" + init_file, rank=rank, world_size=world)
    P = gen.make_problem(n, 3, 1, seed=SEED)
    M = P.M.copy()
    if bad is not None:
        M[bad, bad] = -1.0
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    try:
        ctx = multi.dist_create(n, 3, 1, d(M), d(P.XL), d(P.y), dist=dist, nb=nb)
    except p.GLSError as e:
        np.save(os.path.join(out_dir, "piv%d.npy" % rank), np.array([e.code, e.pivot]))
        dist.destroy_process_group()
        return
    np.save(os.path.join(out_dir, "digest%d.npy" % rank), np.array(multi.shared_state_digest(ctx)))
    lo, hi = multi.snp_range(m, world, rank)
    X = torch.empty((hi - lo, n), dtype=torch.float64, device="cuda")
    p.gen_xr_device(SEED, n, lo, hi - lo, X)
    b = torch.empty((hi - lo, 4), dtype=torch.float64, device="cuda")
    ctx.solve_block(X, hi - lo, b)
    np.save(os.path.join(out_dir, "b%d.npy" % rank), b.cpu().numpy())
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


def _spawn(tmp_path, n, nb, m, bad=None):
    import torch.multiprocessing as mp
    mp.start_processes(_rank_main, args=(2, str(tmp_path / "init"), str(tmp_path), n, nb, m, bad), nprocs=2,
                       join=True, start_method="spawn")


def test_dist_create_two_ranks_matches_oracle(pkg, tmp_path):
    n, nb, m = 1100, 128, 501  # 9 block columns, the last 76 wide: ranks own 5 and 4
    _spawn(tmp_path, n, nb, m)
    np.testing.assert_array_equal(np.load(tmp_path / "digest0.npy"), np.load(tmp_path / "digest1.npy"))
    b = np.concatenate([np.load(tmp_path / "b0.npy"), np.load(tmp_path / "b1.npy")])
    P = gen.make_problem(n, 3, 1, seed=SEED)
    XR = gen.make_XR(SEED, n, 0, m)
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, 1)
    assert_parity(b, np.zeros(m, np.int32), b_or, st_or, label="dist world 2")
    record_parity("dist create world 2 (gloo, one GPU), n=1100 nb=128", b, b_or, st_or)


def test_dist_create_not_spd_pivot(pkg, tmp_path):
    n, nb, bad = 600, 128, 389  # inside block column 3 (owned by rank 1)
    _spawn(tmp_path, n, nb, 10, bad=bad)
    P = gen.make_problem(n, 3, 1, seed=SEED)
    M = P.M.copy()
    M[bad, bad] = -1.0
    with pytest.raises(oracle.NotSPD) as e:
        oracle.cholesky(M)
    for r in (0, 1):
        code, piv = np.load(tmp_path / ("piv%d.npy" % r))
        assert code == 3 and piv == e.value.pivot == bad
