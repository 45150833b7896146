"""Replicate-then-shard through the real library on one GPU.

Two processes, world size 2 over the gloo backend (NCCL refuses two ranks on one device; only one GPU
is available to this build), both on cuda:0: rank 0 runs gls_create, rank 1 gls_create_adopt; the
shared state (packed T, W, G, the int8 digit tiles of T and V, the row scales) is broadcast from
rank 0 with multi.replicate_shared -- the same code bench.py runs over NCCL -- then each rank solves
its own SNP range.  The two shards must equal a single-process solve bit for bit, and rank 1 must have
done its work on the int8 path with the broadcast state.  The ranks' kernels never wait on each other.
"""
import os

import numpy as np
import pytest

import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N, PL, PR, M_PER_RANK = 700, 3, 1, 3000
SEED = 31


def _rank_main(rank, world, init_file, out_dir):
    import torch
    import torch.distributed as dist

    import paper_1210_7325_b200 as pkg
    from paper_1210_7325_b200 import multi

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method="file://" + init_file, rank=rank, world_size=world)
    P = gen.make_problem(N, PL, PR, seed=SEED)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if rank == 0:
        ctx = pkg.Context(N, PL, PR, d(P.M), d(P.XL), d(P.y))
    else:
        ctx = pkg.Context(N, PL, PR, adopt=True)
    # the library's shared buffers broadcast from rank 0 (gloo: staged through host memory)
    multi.replicate_shared(ctx, dist, src=0)
    lo, hi = multi.weak_range(M_PER_RANK, rank)
    X = torch.empty((M_PER_RANK * PR, N), dtype=torch.float64, device="cuda")
    pkg.gen_xr_device(SEED, N, lo * PR, M_PER_RANK * PR, X)
    b = torch.empty((M_PER_RANK, PL + PR), dtype=torch.float64, device="cuda")
    ctx.solve_block(X, M_PER_RANK, b)
    counts = ctx.path_counts()
    np.save(os.path.join(out_dir, "b%d.npy" % rank), b.cpu().numpy())
    np.save(os.path.join(out_dir, "paths%d.npy" % rank), np.array(counts))
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


def test_replicate_then_shard_two_processes(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import paper_1210_7325_b200 as pkg

    init_file = str(tmp_path / "dist_init")
    mp.start_processes(_rank_main, args=(2, init_file, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    b0, b1 = np.load(tmp_path / "b0.npy"), np.load(tmp_path / "b1.npy")
    for r in (0, 1):
        assert tuple(np.load(tmp_path / ("paths%d.npy" % r))) == (1, 0)  # int8 path on both ranks
    # single-process reference over both ranks' SNPs
    P = gen.make_problem(N, PL, PR, seed=SEED)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    X = torch.empty((2 * M_PER_RANK * PR, N), dtype=torch.float64, device="cuda")
    pkg.gen_xr_device(SEED, N, 0, 2 * M_PER_RANK * PR, X)
    with pkg.Context(N, PL, PR, d(P.M), d(P.XL), d(P.y)) as ctx:
        b = torch.empty((2 * M_PER_RANK, PL + PR), dtype=torch.float64, device="cuda")
        ctx.solve_block(X, 2 * M_PER_RANK, b)
        ref = b.cpu().numpy()
    np.testing.assert_array_equal(np.concatenate([b0, b1]), ref)
