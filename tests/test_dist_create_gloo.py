"""NEXT-3 host protocol (multi.dist_create; include/gls.h gls_dist_*) on CPU with gloo, world 1-3.

A numpy stand-in for gls.DistFactor performs the same block algorithm on the rank's column blocks (the
right-looking blocked Cholesky fused with the substitution that turns the identity into T = L^{-1};
dist_create.cu's header), with torch CPU buffers in place of the device ones, and runs through the real
orchestration (panel broadcasts from the block owners, the W all-gather summed in rank order, the
MAX / SUM all-reduces).  Checked: the assembled T equals the inverse of LAPACK's Cholesky factor, W =
T [X_L | y], the row maxima of |T|, every digit-tile byte has exactly its owner's contribution, and a
non-SPD M stops every rank with the same pivot.  The CUDA steps themselves are checked against the
oracle in tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1210_7325_b200 import gls, multi


class FakeDist:
    def __init__(self, n, pL, pR, nb, G, r, M, XL, y):
        self.n, self.nb, self.G, self.r, self.pl1 = n, nb, G, r, pL + 1
        self.nblocks = (n + nb - 1) // nb
        self.own = [j for j in range(self.nblocks) if j % G == r]
        self.A = {j: M[:, j * nb:j * nb + self.w(j)].copy() for j in self.own}   # full-height column blocks
        self.R = {j: np.zeros((n, self.w(j))) for j in self.own}
        self.B = np.column_stack([XL.T, y]) if pL else y[:, None].copy()
        self.panel = torch.zeros(n * nb, dtype=torch.float64)
        self.bufs = {gls.GLS_DIST_WPART: torch.zeros(n * self.pl1, dtype=torch.float64),
                     gls.GLS_DIST_W: torch.zeros(n * self.pl1, dtype=torch.float64),
                     gls.GLS_DIST_ROWMAX: torch.zeros(n, dtype=torch.float64),
                     gls.GLS_DIST_VMAX: torch.zeros(self.pl1, dtype=torch.float64),
                     gls.GLS_DIST_T8: torch.zeros(self.nblocks, dtype=torch.uint8),
                     gls.GLS_DIST_V8: torch.zeros(self.nblocks, dtype=torch.uint8)}
        self.failed_pivot = -1
        self.tol = 2.0 ** -52 * np.max(np.diag(M))

    def w(self, j):
        return min(self.nb, self.n - j * self.nb)

    def buffer(self, which, k=0):
        if which == gls.GLS_DIST_PANEL:
            return self.panel[:(self.n - k * self.nb) * self.w(k)].view(torch.uint8)
        b = self.bufs[which]
        return b if b.dtype == torch.uint8 else b.view(torch.uint8)

    def _panel(self, k):
        ldp = self.n - k * self.nb
        return self.panel[:ldp * self.w(k)].numpy().reshape(self.w(k), ldp).T  # column-major (ldp, w)

    def step(self, phase, k=0):
        n, nb = self.n, self.nb
        if phase == gls.GLS_DIST_FACTOR:
            j0, w = k * nb, self.w(k)
            Akk = self.A[k][j0:j0 + w]
            d = np.linalg.eigvalsh(Akk).min()
            if d <= self.tol:
                self.failed_pivot = j0 + next(i for i in range(1, w + 1)
                                              if np.linalg.eigvalsh(Akk[:i, :i]).min() <= self.tol) - 1
                return gls.GLS_ERR_NOT_SPD
            L = np.linalg.cholesky(Akk)
            T = sla.solve_triangular(L, np.eye(w), lower=True)
            self.R[k][j0:j0 + w] = T
            P = self._panel(k)
            P[:w] = T
            P[w:] = self.A[k][j0 + w:] @ T.T
        elif phase == gls.GLS_DIST_UPDATE:
            j0, w = k * nb, self.w(k)
            P = self._panel(k)
            Tkk, Lb = P[:w], P[w:]
            for j in self.own:
                if j < k:
                    self.R[j][j0:j0 + w] = Tkk @ self.R[j][j0:j0 + w]
                if j <= k:
                    self.R[j][j0 + w:] -= Lb @ self.R[j][j0:j0 + w]
                if j > k:
                    j1 = j * nb
                    Lj = P[j1 - j0:]
                    self.A[j][j1:] -= Lj @ Lj[:self.w(j)].T
        elif phase == gls.GLS_DIST_PARTIALS:
            Wp = sum(self.R[j] @ self.B[j * nb:j * nb + self.w(j)] for j in self.own) if self.own else 0 * self.B
            self.bufs[gls.GLS_DIST_WPART].copy_(torch.from_numpy(np.ascontiguousarray(Wp.T).ravel()))
            rm = np.zeros(n)
            for j in self.own:
                rm = np.maximum(rm, np.abs(self.R[j]).max(axis=1))
            self.bufs[gls.GLS_DIST_ROWMAX].copy_(torch.from_numpy(rm))
        elif phase == gls.GLS_DIST_PACK:
            W = self.bufs[gls.GLS_DIST_W].numpy().reshape(self.pl1, n).T
            vm = np.zeros(self.pl1)
            for j in self.own:
                V = self.R[j][j * nb:].T @ W[j * nb:]
                vm = np.maximum(vm, np.abs(V).max(axis=0))
                self.bufs[gls.GLS_DIST_T8][j] = self.r + 1  # "digit tiles" of the owned chunks
            self.bufs[gls.GLS_DIST_VMAX].copy_(torch.from_numpy(vm))
        elif phase == gls.GLS_DIST_PACK2:
            for j in self.own:
                self.bufs[gls.GLS_DIST_V8][j] = self.r + 1
        return gls.GLS_OK

    def finish(self):
        return self

    def close(self):
        pass


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(n, pL, seed, spd=True):
    rng = np.random.default_rng(seed)
    Z = rng.standard_normal((n, 40))
    M = Z @ Z.T / 40 + np.eye(n)
    if not spd:
        M[n - 5, n - 5] = -1.0
    return M, rng.standard_normal((pL, n)), rng.standard_normal(n)


def _worker(rank, world, port, q, n, nb, spd):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pL = 3
        M, XL, y = _problem(n, pL, 5, spd)
        fd = FakeDist(n, pL, 1, nb, world, rank, M, XL, y)
        try:
            out = multi.dist_create(n, pL, 1, M, XL, y, dist=dist, nb=nb, factor=fd)
        except gls.GLSError as e:
            q.put((rank, "notspd", e.pivot))
            return
        # assemble T from every rank's column blocks
        Tloc = np.zeros((n, n))
        for j in out.own:
            Tloc[:, j * nb:j * nb + out.w(j)] = out.R[j]
        Tt = torch.from_numpy(Tloc)
        dist.all_reduce(Tt)
        W = out.bufs[gls.GLS_DIST_W].numpy().reshape(pL + 1, n).T.copy()
        q.put((rank, "ok", (Tt.numpy(), W, out.bufs[gls.GLS_DIST_ROWMAX].numpy().copy(),
                            out.bufs[gls.GLS_DIST_T8].numpy().copy(), out.bufs[gls.GLS_DIST_V8].numpy().copy())))
    finally:
        dist.destroy_process_group()


def _run(world, n, nb, spd=True):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, n, nb, spd)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,n,nb", [(2, 600, 128), (3, 700, 128), (2, 300, 256)])
def test_dist_create_protocol(world, n, nb):
    res = _run(world, n, nb)
    M, XL, y = _problem(n, 3, 5)
    Tref = sla.solve_triangular(np.linalg.cholesky(M), np.eye(n), lower=True)
    B = np.column_stack([XL.T, y])
    K = (n + nb - 1) // nb
    for rank, kind, (T, W, rm, t8, v8) in res:
        assert kind == "ok"
        np.testing.assert_allclose(T, Tref, rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(W, Tref @ B, rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(rm, np.abs(Tref).max(axis=1), rtol=1e-9)
        assert list(t8) == [j % world + 1 for j in range(K)] and list(v8) == list(t8)
    # every rank holds the same W bits (the rank-order sum)
    for r in res[1:]:
        np.testing.assert_array_equal(r[2][1], res[0][2][1])


def test_dist_create_not_spd_stops_every_rank():
    res = _run(2, 400, 128, spd=False)
    assert all(kind == "notspd" for _, kind, _ in res)
    pivs = {p for _, _, p in res}
    assert len(pivs) == 1 and next(iter(pivs)) <= 400 - 5


def test_dist_create_world1_is_single_process():
    M, XL, y = _problem(333, 3, 5)
    fd = FakeDist(333, 3, 1, 128, 1, 0, M, XL, y)
    out = multi.dist_create(333, 3, 1, M, XL, y, dist=None, nb=128, factor=fd)
    T = np.zeros((333, 333))
    for j in out.own:
        T[:, j * 128:j * 128 + out.w(j)] = out.R[j]
    np.testing.assert_allclose(T, sla.solve_triangular(np.linalg.cholesky(M), np.eye(333), lower=True),
                               rtol=1e-9, atol=1e-11)
