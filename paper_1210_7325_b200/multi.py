"""Replicate-then-shard across GPUs (§6 future work).

The paper's plan for distributed memory: "perform the Cholesky factorization of M redundantly,
and then operate on distinct chunks of X_R".  Here rank 0 factors once (gls_create) and the
shared state -- packed T = L^{-1}, packed [X~_L | y~], and W^T W (S_TL, b_T) -- is broadcast
over NVLink with one NCCL broadcast per buffer (torch.distributed), so every rank holds
bit-identical factors and b is bitwise independent of the number of GPUs.  After that there is
no communication: each rank solves its own contiguous SNP range.

Only host-side plumbing lives here; every arithmetic step runs in libgls.so.
"""
from __future__ import annotations

import os


def snp_range(m_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous problem range [lo, hi) of `rank` when m_total problems are split over `world`
    ranks (strong scaling): floor(r m / G) .. floor((r+1) m / G)."""
    if world < 1 or not (0 <= rank < world) or m_total < 0:
        raise ValueError("bad shard arguments")
    return (rank * m_total) // world, ((rank + 1) * m_total) // world


def local_device(env=None) -> int:
    """CUDA device of this process: LOCAL_RANK (torchrun sets it per node), so the same code runs on
    one node or several -- the SNP shard follows the global rank, the device the local one."""
    env = os.environ if env is None else env
    return int(env.get("LOCAL_RANK", "0"))


def weak_range(m_per_rank: int, rank: int) -> tuple[int, int]:
    """Problem range of `rank` under weak scaling (every rank owns m_per_rank problems)."""
    return rank * m_per_rank, (rank + 1) * m_per_rank


def replicate_shared(ctx, dist, src: int = 0, group=None, int8_only: bool = False) -> int:
    """Broadcast the shared state of `ctx` from rank `src` to every rank of `group`, then commit it
    on the receiving ranks.  `ctx` is a Context created with gls_create on `src` and with
    adopt=True elsewhere.  `src` is a GLOBAL rank (torch.distributed's convention for broadcast).
    Over NCCL the library's device buffers are broadcast in place (zero-copy tensors); over gloo
    (host-only backend, used by the CPU-side tests) they are staged through host memory.
    int8_only: broadcast only the int8 path's state (receivers created with adopt=True, int8_only=True;
    the FP64 path's packed T -- n^2 * 4 bytes -- is neither sent nor allocated on them).
    Returns the number of bytes broadcast."""
    import torch

    from .gls import GLS_SHARE_INT8_ONLY
    rank = dist.get_rank()  # global rank, comparable with src
    tensors = ctx.shared_tensors(GLS_SHARE_INT8_ONLY if int8_only else None)
    staged = bool(tensors) and tensors[0].is_cuda and dist.get_backend(group) == "gloo"
    nbytes = 0
    for t in tensors:
        if staged:
            h = t.cpu()
            dist.broadcast(h, src=src, group=group)
            if rank != src:
                t.copy_(h)
        else:
            dist.broadcast(t, src=src, group=group)
        nbytes += t.numel() * t.element_size()
    if tensors and tensors[0].is_cuda:
        torch.cuda.synchronize()
    if rank != src:
        ctx.commit_shared()
    return nbytes


def max_over_ranks(values, dist, device=None):
    """Element-wise max of a list of floats over all ranks (timings are max-over-ranks)."""
    import torch
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def sum_over_ranks(values, dist, device=None):
    """Element-wise sum of a list of floats over all ranks."""
    import torch
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.cpu()]


def shared_state_digest(ctx) -> list[int]:
    """One 64-bit checksum per shared-state buffer of `ctx` (wrapping sum of its 8-byte words, plus
    a position-weighted sum), computed on the device.  Equal digests on every rank are the evidence
    that redundant per-rank factorisations (the paper's plan) produced the same bits."""
    import torch
    out = []
    for t in ctx.shared_tensors():
        nb = t.numel() - t.numel() % 8
        w = t[:nb].view(torch.int64)
        pos = torch.arange(w.numel(), device=w.device, dtype=torch.int64) % 65521 + 1
        out.append(int(w.sum().item()))
        out.append(int((w * pos).sum().item()))
    return out


class Comm:
    """The collectives of the distributed create over torch.distributed: NCCL moves the library's device
    buffers in place; gloo (host-only, used by the CPU-side and one-GPU tests) stages them through host
    memory.  world 1 (no process group): every collective is the identity."""

    def __init__(self, dist=None, group=None):
        self.dist, self.group = dist, group
        live = dist is not None and dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if live else 1
        self.rank = dist.get_rank(group) if live else 0
        self.host = live and self.world > 1 and dist.get_backend(group) == "gloo"

    def _src(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def _run(self, t, fn):
        if self.world == 1:
            return
        if self.host and t.is_cuda:
            h = t.cpu()
            fn(h)
            t.copy_(h)
        else:
            fn(t)

    def bcast(self, t, src: int):
        self._run(t, lambda x: self.dist.broadcast(x, src=self._src(src), group=self.group))

    def allreduce(self, t, op: str):
        o = {"max": self.dist.ReduceOp.MAX, "sum": self.dist.ReduceOp.SUM}[op] if self.world > 1 else None
        self._run(t, lambda x: self.dist.all_reduce(x, op=o, group=self.group))

    def allgather(self, t):
        if self.world == 1:
            return [t]
        src = t.cpu() if self.host and t.is_cuda else t
        out = [src.new_empty(src.shape) for _ in range(self.world)]
        self.dist.all_gather(out, src, group=self.group)
        return [x.to(t.device) for x in out]


def dist_create(n: int, pL: int, pR: int, M, X_L, y, dist=None, nb: int = 1024, group=None, factor=None):
    """The distributed create of NEXT-3 (include/gls.h gls_dist_*): this rank holds the
    column blocks j of width nb with j % G == rank; one panel broadcast per block column; then the int8
    state assembled by small all-gathers / all-reduces.  Returns this rank's int8-only Context (its shared
    state bit-identical on every rank).  M, X_L, y: full arrays (host or device) -- each rank copies its
    own column blocks of M.  Raises GLSError(GLS_ERR_NOT_SPD) on every rank when a pivot fails (the pivot
    index in the exception's .pivot).  `factor` (tests): a stand-in for gls.DistFactor with the same
    methods."""
    import torch

    from . import gls
    comm = Comm(dist, group)
    d = factor if factor is not None else gls.DistFactor(n, pL, pR, nb, comm.world, comm.rank, M, X_L, y)
    dev = d.buffer(gls.GLS_DIST_W).device
    status = torch.zeros(1, dtype=torch.int64, device=dev)
    for k in range(d.nblocks):
        owner = k % comm.world
        if comm.rank == owner:
            rc = d.step(gls.GLS_DIST_FACTOR, k)
            status[0] = d.failed_pivot if rc == gls.GLS_ERR_NOT_SPD else -1
        comm.bcast(status, owner)
        piv = int(status.item())
        if piv >= 0:
            d.close()
            err = gls.GLSError(gls.GLS_ERR_NOT_SPD, "M is not SPD: Cholesky pivot %d (distributed create)" % piv)
            err.pivot = piv
            raise err
        comm.bcast(d.buffer(gls.GLS_DIST_PANEL, k), owner)
        d.step(gls.GLS_DIST_UPDATE, k)
    d.step(gls.GLS_DIST_PARTIALS)
    parts = comm.allgather(d.buffer(gls.GLS_DIST_WPART).view(torch.float64))
    W = parts[0].clone()
    for p in parts[1:]:  # rank order on every rank: the same bits everywhere
        W += p
    d.buffer(gls.GLS_DIST_W).view(torch.float64).copy_(W)
    comm.allreduce(d.buffer(gls.GLS_DIST_ROWMAX).view(torch.float64), "max")
    d.step(gls.GLS_DIST_PACK)
    comm.allreduce(d.buffer(gls.GLS_DIST_VMAX).view(torch.float64), "max")
    d.step(gls.GLS_DIST_PACK2)
    comm.allreduce(d.buffer(gls.GLS_DIST_T8), "sum")  # uint8 bytes, one nonzero contributor each
    comm.allreduce(d.buffer(gls.GLS_DIST_V8), "sum")
    if dev.type == "cuda":
        torch.cuda.synchronize()
    ctx = d.finish()
    d.close()
    return ctx
