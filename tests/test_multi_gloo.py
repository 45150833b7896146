"""Multi-process (gloo, world size 2, CPU) tests of the replicate-then-shard host protocol
(paper_1210_7325_b200/multi.py).  The CUDA kernels are exercised by the GPU
tests; here a stand-in context with CPU buffers checks that the broadcast reproduces the root's
shared state bit for bit, that only non-root ranks commit, that shards tile [0, m) exactly and
that timings reduce to the max over ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1210_7325_b200.multi import local_device, max_over_ranks, replicate_shared, snp_range, weak_range


class FakeCtx:
    """Stands in for gls.Context: CPU shared buffers, commit flag."""

    def __init__(self, root: bool):
        g = torch.Generator().manual_seed(1234)
        sizes = [4096 * 8, 1024 * 8, 16 * 8]
        if root:
            self.bufs = [torch.randint(0, 256, (s,), dtype=torch.uint8, generator=g) for s in sizes]
        else:
            self.bufs = [torch.zeros(s, dtype=torch.uint8) for s in sizes]
        self.committed = root

    def shared_tensors(self, flags=None):
        return self.bufs

    def commit_shared(self):
        assert not self.committed, "commit called twice or on root"
        self.committed = True


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = FakeCtx(root=(rank == 0))
        nbytes = replicate_shared(ctx, dist, src=0)
        ref = FakeCtx(root=True)
        same = all(torch.equal(a, b) for a, b in zip(ctx.bufs, ref.bufs))
        t = max_over_ranks([float(rank + 1), 10.0 - rank], dist)
        lo, hi = snp_range(1_000_003, world, rank)
        q.put((rank, same, ctx.committed, nbytes, t, lo, hi))
    finally:
        dist.destroy_process_group()


def test_replicate_and_shard_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, committed, nbytes, t, lo, hi in res:
        assert same and committed
        assert nbytes == 4096 * 8 + 1024 * 8 + 16 * 8
        assert t == [2.0, 10.0]
    assert res[0][5] == 0 and res[0][6] == res[1][5] and res[1][6] == 1_000_003


@pytest.mark.parametrize("m,world", [(0, 1), (1, 2), (7, 3), (1_000_000, 8), (220_833, 8)])
def test_snp_range_tiles(m, world):
    got = [snp_range(m, world, r) for r in range(world)]
    assert got[0][0] == 0 and got[-1][1] == m
    for (a, b), (c, d) in zip(got, got[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in got]
    assert max(sizes) - min(sizes) <= 1


def test_weak_range():
    assert weak_range(1_000_000, 0) == (0, 1_000_000)
    assert weak_range(1_000_000, 7) == (7_000_000, 8_000_000)
    with pytest.raises(ValueError):
        snp_range(10, 2, 2)


def _worker_2x2(rank, world, port, q):
    """One rank of a 2-node x 2-GPU layout as torchrun --nnodes 2 --nproc-per-node 2 sets it up."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["LOCAL_RANK"] = str(rank % 2)
    os.environ["LOCAL_WORLD_SIZE"] = "2"
    os.environ["GROUP_RANK"] = str(rank // 2)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = FakeCtx(root=(rank == 0))
        replicate_shared(ctx, dist, src=0)
        ref = FakeCtx(root=True)
        same = all(torch.equal(a, b) for a, b in zip(ctx.bufs, ref.bufs))
        t = max_over_ranks([float(rank)], dist)
        q.put((rank, same, ctx.committed, local_device(), weak_range(1000, rank), t))
    finally:
        dist.destroy_process_group()


def test_replicate_and_shard_two_nodes_gloo():
    """NEXT-3 host side: the protocol spans nodes unchanged -- rank 0 on node 0 broadcasts to the
    ranks of both nodes, every rank's device is its LOCAL_RANK, its SNP shard follows its global
    rank, and timings reduce over all four ranks."""
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_2x2, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, committed, dev, rng, t in res:
        assert same and committed
        assert dev == rank % 2
        assert rng == (1000 * rank, 1000 * (rank + 1))
        assert t == [3.0]


def test_local_device_env():
    assert local_device({}) == 0
    assert local_device({"LOCAL_RANK": "3"}) == 3


def _worker_subgroup(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grp = dist.new_group([1, 2])
        if rank in (1, 2):
            # the subgroup's root is GLOBAL rank 1 (group rank 0): it must not commit, rank 2 must
            ctx = FakeCtx(root=(rank == 1))
            replicate_shared(ctx, dist, src=1, group=grp)
            ref = FakeCtx(root=True)
            same = all(torch.equal(a, b) for a, b in zip(ctx.bufs, ref.bufs))
            q.put((rank, same, ctx.committed))
        else:
            q.put((rank, True, True))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_replicate_in_subgroup_rooted_at_global_rank_1():
    """src is a global rank: in a subgroup {1, 2} rooted at global rank 1, rank 1 keeps its state
    (no commit) and rank 2 receives it and commits (group-local vs global rank)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_subgroup, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(same and committed for _, same, committed in res), res
