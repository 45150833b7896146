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


def replicate_shared(ctx, dist, src: int = 0, group=None) -> int:
    """Broadcast the shared state of `ctx` from rank `src` to every rank of `group`, then commit it
    on the receiving ranks.  `ctx` is a Context created with gls_create on `src` and with
    adopt=True elsewhere.  `src` is a GLOBAL rank (torch.distributed's convention for broadcast).
    Over NCCL the library's device buffers are broadcast in place (zero-copy tensors); over gloo
    (host-only backend, used by the CPU-side tests) they are staged through host memory.
    Returns the number of bytes broadcast."""
    import torch
    rank = dist.get_rank()  # global rank, comparable with src
    tensors = ctx.shared_tensors()
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
