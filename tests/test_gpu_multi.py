"""Replicate-then-shard through the real library on one GPU.

Two processes, world size 2 over the gloo backend (NCCL refuses two ranks on one device; only one GPU
is available to this build), both on cuda:0.  Two ways to replicate the shared state:
  bcast     -- rank 0 runs gls_create, rank 1 gls_create_adopt; the shared state (packed T, W, G, the
               int8 digit tiles of T and V, the row scales) is broadcast from rank 0 with
               multi.replicate_shared (the code bench.py runs with --replicate bcast);
  redundant -- every rank runs gls_create itself (the paper's "factorization of M redundantly",
               PAPER.md:812-814; bench.py's default), and the shared-state digests must agree.
Then each rank solves its strong-scaling shard multi.snp_range(m, 2, rank) of an odd m.  The two
shards must equal a single-process solve of all m problems bit for bit, and both ranks must have done
their work on the int8 path.  The ranks' kernels never wait on each other.
"""
import os

import numpy as np
import pytest

import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N, PL, PR, M_TOTAL = 700, 3, 1, 6001
SEED = 31


def _rank_main(rank, world, init_file, out_dir, mode):
    import torch
    import torch.distributed as dist

    import paper_1210_7325_b200 as pkg
    from paper_1210_7325_b200 import multi

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method="file://" + init_file, rank=rank, world_size=world)
    P = gen.make_problem(N, PL, PR, seed=SEED)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if mode in ("bcast", "bcast8"):
        i8 = mode == "bcast8"  # receivers hold only the int8 path's state; the root sends only that
        ctx = (pkg.Context(N, PL, PR, d(P.M), d(P.XL), d(P.y)) if rank == 0
               else pkg.Context(N, PL, PR, adopt=True, int8_only=i8))
        # the library's shared buffers broadcast from rank 0 (gloo: staged through host memory)
        nbytes = multi.replicate_shared(ctx, dist, src=0, int8_only=i8)
        full = sum(nb for _, nb in ctx.shared_view(0)) if rank == 0 else 0
        np.save(os.path.join(out_dir, "nbytes%d.npy" % rank), np.array([nbytes, full]))
    else:
        ctx = pkg.Context(N, PL, PR, d(P.M), d(P.XL), d(P.y))
    np.save(os.path.join(out_dir, "digest%d.npy" % rank),
            np.array(multi.shared_state_digest(ctx) if mode != "bcast8" else [0]))
    lo, hi = multi.snp_range(M_TOTAL, world, rank)
    X = torch.empty((hi - lo) * PR, N, dtype=torch.float64, device="cuda")
    pkg.gen_xr_device(SEED, N, lo * PR, (hi - lo) * PR, X)
    b = torch.empty((hi - lo, PL + PR), dtype=torch.float64, device="cuda")
    ctx.solve_block(X, hi - lo, b)
    counts = ctx.path_counts()
    np.save(os.path.join(out_dir, "b%d.npy" % rank), b.cpu().numpy())
    np.save(os.path.join(out_dir, "paths%d.npy" % rank), np.array(counts))
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["bcast", "bcast8", "redundant"])
def test_replicate_then_shard_two_processes(tmp_path, mode):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import paper_1210_7325_b200 as pkg

    init_file = str(tmp_path / "dist_init")
    mp.start_processes(_rank_main, args=(2, init_file, str(tmp_path), mode), nprocs=2, join=True,
                       start_method="spawn")
    b0, b1 = np.load(tmp_path / "b0.npy"), np.load(tmp_path / "b1.npy")
    assert len(b0) == M_TOTAL // 2 and len(b1) == M_TOTAL - M_TOTAL // 2
    for r in (0, 1):
        assert tuple(np.load(tmp_path / ("paths%d.npy" % r))) == (1, 0)  # int8 path on both ranks
    np.testing.assert_array_equal(np.load(tmp_path / "digest0.npy"), np.load(tmp_path / "digest1.npy"))
    if mode == "bcast8":  # only T8, aux, V8, vscale and G travel: no packed FP64 T
        sent, full = np.load(tmp_path / "nbytes0.npy")
        assert sent == np.load(tmp_path / "nbytes1.npy")[0] and sent < 0.6 * full, (sent, full)
    # single-process reference over all m problems
    P = gen.make_problem(N, PL, PR, seed=SEED)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    X = torch.empty((M_TOTAL * PR, N), dtype=torch.float64, device="cuda")
    pkg.gen_xr_device(SEED, N, 0, M_TOTAL * PR, X)
    with pkg.Context(N, PL, PR, d(P.M), d(P.XL), d(P.y)) as ctx:
        b = torch.empty((M_TOTAL, PL + PR), dtype=torch.float64, device="cuda")
        ctx.solve_block(X, M_TOTAL, b)
        ref = b.cpu().numpy()
    np.testing.assert_array_equal(np.concatenate([b0, b1]), ref)
