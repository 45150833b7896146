"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, on the same seeded inputs.

Every input comes from gen/ (CPU) or its independent device twin (libglsgen_dev.so, checked
bit-exact here first); every expected value comes from oracle/.  Tolerance: the north-star
1e-9 per b_i entry, guarded as in DESIGN.md reading A10 (tests/_util.py).
"""
import os

import numpy as np
import pytest

import gen
import oracle

from _util import assert_parity, edge_set, int8_chunk_bounds, normwise_err, record_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = gen.DEFAULT_SEED


@pytest.fixture(scope="module")
def glsmod():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1210_7325_b200 as pkg
    pkg.load()
    return pkg


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_gpu(pkg, P, XR_dev, m, pR, host_out=False, status=True, path=None, counts=None):
    p = P.pL + pR
    ctx = pkg.Context(P.n, P.pL, pR, dev(P.M), dev(P.XL) if P.pL else None, dev(P.y))
    try:
        if path is not None:
            ctx.set_path(path)
        if host_out:
            b = np.empty((m, p))
            st = np.empty(m, dtype=np.int32)
        else:
            b = torch.empty((m, p), dtype=torch.float64, device="cuda")
            st = torch.empty(m, dtype=torch.int32, device="cuda")
        ctx.solve_block(XR_dev, m, b, st if status else None)
        launches = ctx.kernel_launches
        if counts is not None:
            counts.extend(ctx.path_counts())
    finally:
        ctx.close()
    if not host_out:
        b, st = b.cpu().numpy(), st.cpu().numpy()
    return b, st, launches


def test_device_generator_matches_cpu(glsmod):
    for n, col0, ncols in [(500, 0, 37), (1501, 12345, 9), (10_000, 999_990, 3)]:
        X = torch.empty((ncols, n), dtype=torch.float64, device="cuda")
        glsmod.gen_xr_device(SEED, n, col0, ncols, X)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(X.cpu().numpy(), gen.make_XR(SEED, n, col0, ncols))


def test_config0_all_snps(glsmod):
    """Config 0 (n=500, pL=3, pR=1, m=2000): every SNP against the oracle."""
    cfg = gen.CONFIGS[0]
    P = gen.config_problem(cfg)
    XR = gen.make_XR(SEED, cfg.n, 0, cfg.cols)
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, cfg.pR)
    Xd = torch.empty((cfg.cols, cfg.n), dtype=torch.float64, device="cuda")
    glsmod.gen_xr_device(SEED, cfg.n, 0, cfg.cols, Xd)
    b, st, launches = run_gpu(glsmod, P, Xd, cfg.m, cfg.pR)
    assert launches > 0
    assert_parity(b, st, b_or, st_or, label="config0")
    assert normwise_err(b, b_or) <= 1e-12
    record_parity("config0 n=500 p=4: every SNP", b, b_or, st_or)


@pytest.mark.parametrize("n,pL,pR,m,sex", [
    (37, 3, 1, 70, True),       # n < 128: one row block, ragged rows; odd n -> staged path
    (130, 0, 1, 65, False),     # pL = 0: pure X_R regression
    (256, 1, 2, 200, False),    # exact multiple of 128
    (300, 7, 1, 129, True),     # pL + 1 = 8: one full W tile
    (300, 8, 1, 100, True),     # pL + 1 = 9: two W tiles
    (420, 16, 4, 50, False),    # config-3 shape (p = 20), 2 W tiles... 17 columns -> 3 tiles
    (333, 2, 3, 77, True),      # pR = 3: groups straddle 8-column MMA tiles (full Gram)
    (200, 0, 20, 9, False),     # pR = 20, p = 20
    (515, 4, 5, 41, True),      # pR = 5
    (640, 3, 8, 33, True),      # pR = 8
    (771, 19, 1, 40, False),    # p = 20 with pL = 19 (3 W tiles)
    (2, 0, 1, 50, False),       # smallest problem: n = 2, p = 1
    (21, 19, 1, 33, False),     # p = 20 with n = p + 1
    (160, 2, 16, 5, True),      # pR = 16: two groups per warp quadrant
])
def test_ragged_shapes(glsmod, n, pL, pR, m, sex):
    """Both arithmetic paths (int8 digit split on tcgen05, FP64 DMMA) against the oracle."""
    P = gen.make_problem(n, pL, pR, with_sex=sex, seed=SEED + n)
    XR = gen.make_XR(SEED + n, n, 0, m * pR)
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
    for path, want in ((glsmod.GLS_PATH_AUTO, 0), (glsmod.GLS_PATH_FP64, 1)):
        counts = []
        b, st, _ = run_gpu(glsmod, P, dev(XR), m, pR, path=path, counts=counts)
        assert counts[want] >= 1 and counts[1 - want] == 0, counts
        assert_parity(b, st, b_or, st_or, label="n=%d pL=%d pR=%d path=%d" % (n, pL, pR, path))


def test_non_integer_block_falls_back_to_fp64(glsmod):
    """Imputed dosages (non-integer X_R) are not int8-representable: AUTO must run the FP64 kernel
    for them, decided on the device, and still match the oracle.  The path is chosen per problem: a
    single non-integer value sends only its own problem to the FP64 kernel -- that row equals the FP64
    path's bit for bit, every other row the all-integer int8 run's."""
    n, pL, pR, m = 700, 3, 1, 300
    P = gen.make_problem(n, pL, pR, seed=21)
    XR = gen.make_XR(21, n, 0, m)
    XR = XR + 0.25 * (np.arange(XR.size).reshape(XR.shape) % 3 == 0)  # dosage-like fractions
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
    counts = []
    b, st, _ = run_gpu(glsmod, P, dev(XR), m, pR, counts=counts)
    assert counts == [0, 1], counts
    assert_parity(b, st, b_or, st_or, label="dosage fallback")
    # edge values of the int8 test: out of range, the int8 extremes, -0.0, a fraction in the last
    # row of the last column
    b_int, _, _ = run_gpu(glsmod, P, dev(gen.make_XR(21, n, 0, m)), m, pR)
    for (i, r, v, fallback) in ((5, 17, 200.0, True), (5, 17, -128.0, False), (5, 17, 127.0, False),
                                (5, 17, 128.0, True), (m - 1, n - 1, 1.5, True), (0, 0, -0.0, False),
                                (3, 3, 1e-300, True), (3, 3, float("inf"), True)):
        XR2 = gen.make_XR(21, n, 0, m)
        XR2[i, r] = v
        counts = []
        b2, st2, _ = run_gpu(glsmod, P, dev(XR2), m, pR, counts=counts)
        assert counts == ([1, 1] if fallback else [1, 0]), (i, r, v, counts)
        others = np.arange(m) != i
        np.testing.assert_array_equal(b2[others], b_int[others])
        if fallback:
            b64, _, _ = run_gpu(glsmod, P, dev(XR2), m, pR, path=glsmod.GLS_PATH_FP64)
            np.testing.assert_array_equal(b2[i], b64[i])
        if np.isfinite(v):
            b_or2, st_or2 = oracle.solve(P.M, P.XL, P.y, XR2, pR)
            assert_parity(b2, st2, b_or2, st_or2, label="value %g" % v)


def test_mixed_chunks_pick_paths_independently(glsmod):
    """A device block spanning two int8 conversion chunks (one wave of tiles, then up to 8 waves):
    the integer chunk runs on int8, the chunk holding a dosage runs on FP64; all rows match."""
    n, pL, pR = 64, 2, 1
    chunk = 148 * 128 * 8
    m = chunk + 5000
    P = gen.make_problem(n, pL, pR, seed=22)
    XR = gen.make_XR(22, n, 0, m)
    XR[chunk + 123, 9] = 0.5
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
    counts = []
    b, st, _ = run_gpu(glsmod, P, dev(XR), m, pR, counts=counts)
    # every chunk ran on int8; the dosage's chunk also ran the FP64 kernel, for that one problem
    assert counts[0] >= 2 and counts[1] == 1, counts
    assert_parity(b, st, b_or, st_or, label="mixed chunks")
    XRi = XR.copy()
    XRi[chunk + 123, 9] = 0.0
    b_int, _, _ = run_gpu(glsmod, P, dev(XRi), m, pR)
    others = np.arange(m) != chunk + 123
    np.testing.assert_array_equal(b[others], b_int[others])


@pytest.mark.parametrize("n,pL,pR,m", [(1200, 3, 2, 5000), (1100, 16, 4, 1500)])
def test_path_choice_is_per_problem_and_partition_independent(glsmod, n, pL, pR, m):
    """SPEC's invariant that b is bitwise independent of the block partition holds for mixed data too:
    non-integer problems scattered over a block (some in the same tile as integer ones, groups with one
    bad column) give the same bits whether the block is solved in one call, split at ragged points, or
    streamed from host memory in small host chunks; flagged rows equal the FP64 path's.  p = 20 takes the
    int8 kernel's separate posv (records in a workspace), which must skip the flagged problems too."""
    P = gen.make_problem(n, pL, pR, seed=77)
    XR = gen.make_XR(77, n, 0, m * pR)
    bad_groups = sorted({g for g in (0, 1, 130, 131, 1023, 1024, 2047, 2048) if g < m} | {m - 1})
    for g in bad_groups:
        XR[g * pR + (g % 2), (37 * g) % n] += 0.5
    Xd = dev(XR)
    b_one, st_one, _ = run_gpu(glsmod, P, Xd, m, pR)
    b64, _, _ = run_gpu(glsmod, P, Xd, m, pR, path=glsmod.GLS_PATH_FP64)
    np.testing.assert_array_equal(b_one[bad_groups], b64[bad_groups])
    b_int, _, _ = run_gpu(glsmod, P, dev(np.rint(XR)), m, pR)
    good = np.setdiff1d(np.arange(m), bad_groups)
    np.testing.assert_array_equal(b_one[good], b_int[good])
    with glsmod.Context(n, pL, pR, dev(P.M), dev(P.XL), dev(P.y)) as ctx:
        for cuts in ((1, m // 2 - 1), (131, m - 1), (m // 7, m // 2, 3 * m // 5)):
            b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
            edges = [0, *cuts, m]
            for g0, g1 in zip(edges[:-1], edges[1:]):
                ctx.solve_block(Xd[g0 * pR:g1 * pR], g1 - g0, b[g0:g1])
            np.testing.assert_array_equal(b.cpu().numpy(), b_one)
        Xh = torch.from_numpy(XR).pin_memory()
        bh = torch.empty((m, pL + pR), dtype=torch.float64, pin_memory=True)
        ctx.set_block_cols(640)
        ctx.solve_block(Xh, m, bh)
        np.testing.assert_array_equal(bh.numpy(), b_one)
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR[np.repeat(np.array(bad_groups) * pR, pR) +
                                                  np.tile(np.arange(pR), len(bad_groups))], pR)
    assert_parity(b_one[bad_groups], st_one[bad_groups], b_or, st_or, label="per-problem FP64 rows")


@pytest.mark.parametrize("n", [4096, 4097])
def test_convert_ahead_chunks(glsmod, n):
    """n >= 4096: every chunk of a block after the first is converted to int8 by the convert-ahead
    warps of the previous chunk's kernel (also when that kernel is gated off).  n = 4096 takes the
    in-place device path; odd n = 4097 the staged one (blocks of 4 waves, ld = n + 1) and leaves a
    one-row piece at the end of every column (read directly, not by bulk copy).  A non-integer value
    in the last row of a column in chunk 1 or 2 of a block (1, 2, 1 waves) sends exactly that chunk
    to the FP64 kernel; all rows agree with the FP64 path, and sampled SNPs with the oracle."""
    pL, pR = 2, 1
    w = 148 * 128                       # SNPs per wave of tiles (pR = 1)
    m = 6 * w - 777                     # several chunks, ragged last one
    P = gen.make_problem(n, pL, pR, seed=41)
    Xd = torch.empty((m, n), dtype=torch.float64, device="cuda")
    for c in range(0, m, 16384):
        k = min(16384, m - c)
        glsmod.gen_xr_device(41, n, c, k, Xd[c:c + k])
    counts0 = []
    b, st, _ = run_gpu(glsmod, P, Xd, m, pR, counts=counts0)
    assert counts0[1] == 0 and counts0[0] >= 3, counts0
    b64, st64, _ = run_gpu(glsmod, P, Xd, m, pR, path=glsmod.GLS_PATH_FP64)
    assert_parity(b, st, b64, st64, label="int8 vs FP64 path")
    for col, value in ((w + 1234, 0.5), (3 * w + 1234, 128.0)):  # chunk 1 and chunk 2 of the first block
        Xd2 = Xd.clone()
        Xd2[col, n - 1] = value
        counts = []
        b2, st2, _ = run_gpu(glsmod, P, Xd2, m, pR, counts=counts)
        assert counts == [counts0[0], 1], (col, value, counts, counts0)
        b64, st64, _ = run_gpu(glsmod, P, Xd2, m, pR, path=glsmod.GLS_PATH_FP64)
        assert_parity(b2, st2, b64, st64, label="int8 vs FP64 path, value %g" % value)
        # per-problem path: only the touched problem ran on FP64 (its bits are the FP64 path's)
        others = np.arange(m) != col
        np.testing.assert_array_equal(b2[others], b[others])
        np.testing.assert_array_equal(b2[col], b64[col])
        del Xd2
    # oracle on SNPs around the chunk boundaries and the ragged end
    pick = sorted({0, 1, m - 1, m - 2} | {x + d for x in (w, 3 * w, 4 * w, 5 * w) for d in (-1, 0)})
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, Xd[pick].cpu().numpy(), pR)
    assert_parity(b[pick], st[pick], b_or, st_or, label="convert-ahead vs oracle")


@pytest.mark.parametrize("n,pL,pR,m", [(4100, 0, 20, 2500), (5000, 19, 1, 70000)])
def test_large_p_with_convert_ahead(glsmod, n, pL, pR, m):
    """p = 20 at n >= 4096: the 21-accumulator kernels, the separate batched posv (p > 8) and the
    convert-ahead chunks together.  All rows against the FP64 path, sampled groups against the
    oracle."""
    P = gen.make_problem(n, pL, pR, seed=43)
    cols = m * pR
    Xd = torch.empty((cols, n), dtype=torch.float64, device="cuda")
    for c in range(0, cols, 16384):
        k = min(16384, cols - c)
        glsmod.gen_xr_device(43, n, c, k, Xd[c:c + k])
    counts = []
    b, st, _ = run_gpu(glsmod, P, Xd, m, pR, counts=counts)
    assert counts[1] == 0 and counts[0] >= 3, counts  # int8 only, several chunks
    b64, st64, _ = run_gpu(glsmod, P, Xd, m, pR, path=glsmod.GLS_PATH_FP64)
    assert_parity(b, st, b64, st64, label="int8 vs FP64 path")
    pick = [0, 1, m // 3, m // 2, m - 2, m - 1]
    XR = torch.cat([Xd[g * pR:(g + 1) * pR] for g in pick]).cpu().numpy()
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
    assert_parity(b[pick], st[pick], b_or, st_or, label="vs oracle")


def test_host_stream_equals_device_bitwise(glsmod):
    """Host-resident X_R (Alg. 8 double-buffered stream) gives the same bits as device X_R,
    for several block sizes (block-partition independence)."""
    n, pL, pR, m = 512, 3, 1, 1000
    P = gen.make_problem(n, pL, pR, seed=3)
    XR = gen.make_XR(3, n, 0, m)
    ctx = glsmod.Context(n, pL, pR, dev(P.M), dev(P.XL), dev(P.y))
    try:
        bd = torch.empty((m, 4), dtype=torch.float64, device="cuda")
        ctx.solve_block(dev(XR), m, bd)
        ref = bd.cpu().numpy()
        XRh = torch.from_numpy(XR).pin_memory()
        for cols in (64, 100, 333, 10_000):
            ctx.set_block_cols(cols)
            bh = np.empty((m, 4))
            sth = np.empty(m, dtype=np.int32)
            ctx.solve_block(XRh, m, bh, sth)
            np.testing.assert_array_equal(bh, ref)
            assert np.all(sth == 0)
        # pageable numpy input, host output
        bh = np.empty((m, 4))
        ctx.solve_block(XR, m, bh)
        np.testing.assert_array_equal(bh, ref)
        # split into sub-blocks through the device path
        for cut in (1, 63, 64, 65, 500):
            b1 = torch.empty((cut, 4), dtype=torch.float64, device="cuda")
            b2 = torch.empty((m - cut, 4), dtype=torch.float64, device="cuda")
            Xd = dev(XR)
            ctx.solve_block(Xd[:cut], cut, b1)
            ctx.solve_block(Xd[cut:], m - cut, b2)
            np.testing.assert_array_equal(torch.cat([b1, b2]).cpu().numpy(), ref)
    finally:
        ctx.close()


def test_stream_report_accounts_every_chunk(glsmod):
    """Overlap accounting of the host -> HBM stream (Alg. 8): every chunk of every streamed call is
    reported, the byte counts are exact, the engine times fit inside the wall time, and the
    accounting changes no bit of b."""
    n, pL, pR, m = 2048, 3, 1, 20000
    P = gen.make_problem(n, pL, pR, seed=27)
    XR = gen.make_XR(27, n, 0, m)
    XRh = torch.from_numpy(XR).pin_memory()
    G = torch.from_numpy(XR.astype(np.int8)).pin_memory()
    with glsmod.Context(n, pL, pR, dev(P.M), dev(P.XL), dev(P.y)) as ctx:
        ref = torch.empty((m, 4), dtype=torch.float64, device="cuda")
        ctx.solve_block(dev(XR), m, ref)
        ref = ref.cpu()
        ctx.set_block_cols(3000)
        ctx.set_stream_report(True)
        for label, fn, esz in (("f64", lambda bh, sh: ctx.solve_block(XRh, m, bh, sh), 8),
                               ("i8", lambda bh, sh: ctx.solve_block_i8(G, m, bh, sh), 1)):
            bh = torch.empty((m, 4), dtype=torch.float64).pin_memory()
            sh = torch.empty(m, dtype=torch.int32).pin_memory()
            fn(bh, sh)
            r = ctx.read_stream_report()
            assert torch.equal(bh, ref), label
            nch = (m + 2999) // 3000 if label == "f64" else 1 + (m - 750 + 2999) // 3000  # i8: quarter first chunk
            assert r["chunks"] == nch, (label, r)
            assert r["h2d_bytes"] == m * n * esz and r["d2h_bytes"] == m * (4 * 8 + 4), (label, r)
            busy = r["compute_ms"] + r["first_load_ms"] + r["exposed_h2d_ms"] + r["exposed_other_ms"] + r["tail_ms"]
            assert r["wall_ms"] > 0 and abs(busy - r["wall_ms"]) <= 1e-3 * r["wall_ms"] + 0.05, (label, r)
            assert min(r["first_load_ms"], r["exposed_h2d_ms"], r["exposed_other_ms"], r["tail_ms"]) >= 0, r
            assert r["h2d_ms"] <= r["wall_ms"] and r["compute_ms"] <= r["wall_ms"], r
        assert ctx.read_stream_report()["chunks"] == 0  # the read resets


@pytest.mark.parametrize("piv", [5, 100, 200, 260, 299])
def test_not_spd_pivot_matches_oracle(glsmod, piv):
    """The first failing pivot, wherever it falls: a 64-row leaf, the first or the second sweep of a
    fused 65-128-row node (n = 300 splits 192 = 128 + 64, then 108 = 64 + 44), the last row."""
    n = 300
    P = gen.make_problem(n, 3, 1, seed=4)
    M = P.M.copy()
    M[piv, piv] = -1.0  # the first piv pivots fine, pivot piv negative
    with pytest.raises(oracle.NotSPD) as ei:
        oracle.cholesky(M)
    with pytest.raises(glsmod.GLSError) as eg:
        glsmod.Context(n, 3, 1, dev(M), dev(P.XL), dev(P.y))
    assert eg.value.code == 3
    ctx_pivot = None
    # failed pivot is reported through the ABI
    import ctypes
    L = glsmod.load()
    h = ctypes.c_void_p()
    Md, XLd, yd = dev(M), dev(P.XL), dev(P.y)  # keep the tensors alive across the raw calls
    rc = L.gls_create(n, 3, 1, Md.data_ptr(), XLd.data_ptr(), yd.data_ptr(), ctypes.byref(h))
    assert rc == 3 and h.value
    ctx_pivot = L.gls_failed_pivot(h)
    assert L.gls_solve_block(h, yd.data_ptr(), 1, yd.data_ptr()) == 6  # GLS_ERR_STATE
    L.gls_destroy(h)
    assert ctx_pivot == ei.value.pivot == piv


def test_rank_deficient_isolation(glsmod):
    n, m = 400, 130
    P = gen.make_problem(n, 3, 1, with_sex=True, seed=5)
    XR = gen.make_XR(5, n, 0, m)
    XR[7] = 0.0
    XR[64] = 2.0 * P.XL[2]
    XR[129] = 0.0
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, 1)
    assert list(np.nonzero(st_or)[0]) == [7, 64, 129]
    b, st, _ = run_gpu(glsmod, P, dev(XR), m, 1)
    assert_parity(b, st, b_or, st_or, label="rank-deficient")


def test_scaling_invariance_bitwise(glsmod):
    """b(4M) == b(M) bit for bit on the GPU (all arithmetic scales by exact powers of 2)."""
    n, m = 384, 300
    P = gen.make_problem(n, 3, 1, seed=6)
    Xd = dev(gen.make_XR(6, n, 0, m))
    b1, _, _ = run_gpu(glsmod, P, Xd, m, 1)
    P4 = gen.Problem(P.n, P.pL, P.pR, 4.0 * P.M, P.XL, P.y, P.beta_L)
    b4, _, _ = run_gpu(glsmod, P4, Xd, m, 1)
    np.testing.assert_array_equal(b1, b4)


def test_planted_beta_config1_all_snps(glsmod):
    """Full config 1 size (n=1500, m=220833), noise-free y = X_L beta: b_i = (beta, 0) for all i."""
    cfg = gen.CONFIGS[1]
    P = gen.config_problem(cfg, noise=0.0)
    Xd = torch.empty((cfg.cols, cfg.n), dtype=torch.float64, device="cuda")
    glsmod.gen_xr_device(SEED, cfg.n, 0, cfg.cols, Xd)
    b, st, _ = run_gpu(glsmod, P, Xd, cfg.m, cfg.pR)
    assert np.all(st == 0)
    ref = np.concatenate([P.beta_L, [0.0]])
    err = np.max(np.abs(b - ref)) / np.max(np.abs(P.beta_L))
    assert err <= 1e-10, err


def test_config1_all_snps(glsmod):
    """Config 1 at full size (n=1500, m=220833) in the bench launch configuration (one device block):
    EVERY SNP against the oracle (SURVEY §8(c) coverage plan), X_R for the oracle drawn on the CPU."""
    cfg = gen.CONFIGS[1]
    P = gen.config_problem(cfg)
    Xd = torch.empty((cfg.cols, cfg.n), dtype=torch.float64, device="cuda")
    glsmod.gen_xr_device(SEED, cfg.n, 0, cfg.cols, Xd)
    b, st, _ = run_gpu(glsmod, P, Xd, cfg.m, cfg.pR)
    del Xd
    XR = gen.make_XR(SEED, cfg.n, 0, cfg.cols)
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, cfg.pR)
    assert_parity(b, st, b_or, st_or, label="config1 all SNPs")
    record_parity("config1 n=1500 p=4: all 220833 SNPs", b, b_or, st_or)
    # the FP64 DMMA path on the same inputs, every SNP
    b64, st64, _ = run_gpu(glsmod, P, dev(XR), cfg.m, cfg.pR, path=glsmod.GLS_PATH_FP64)
    assert_parity(b64, st64, b_or, st_or, label="config1 all SNPs, FP64 path")
    record_parity("config1, FP64 DMMA path: all 220833 SNPs", b64, b_or, st_or)


def test_adopt_shared_state_bitwise(glsmod):
    """Replicate-then-shard: an adopt-mode context fed the root's shared buffers (what the NCCL
    broadcast delivers) solves bit-identically."""
    n, m = 300, 200
    P = gen.make_problem(n, 3, 1, seed=8)
    Xd = dev(gen.make_XR(8, n, 0, m))
    root = glsmod.Context(n, 3, 1, dev(P.M), dev(P.XL), dev(P.y))
    other = glsmod.Context(n, 3, 1, adopt=True)
    try:
        with pytest.raises(glsmod.GLSError):
            other.solve_block(Xd, m, torch.empty((m, 4), dtype=torch.float64, device="cuda"))
        for src, dst in zip(root.shared_tensors(), other.shared_tensors()):
            assert src.numel() == dst.numel()
            dst.copy_(src)
        torch.cuda.synchronize()
        other.commit_shared()
        b1 = torch.empty((m, 4), dtype=torch.float64, device="cuda")
        b2 = torch.empty((m, 4), dtype=torch.float64, device="cuda")
        root.solve_block(Xd, m, b1)
        other.solve_block(Xd, m, b2)
        assert torch.equal(b1, b2)
    finally:
        root.close()
        other.close()


@pytest.fixture(scope="module")
def n1e4_factor():
    """Oracle Cholesky of the n = 1e4 M of configs 2-4 (computed once, ~10 s on 16 cores)."""
    P = gen.config_problem(gen.CONFIGS[2])
    return P, oracle.cholesky(P.M)


def test_config2_full_size_sampled_parity_and_planted_beta(glsmod, n1e4_factor):
    """Config 2 at full size (n=1e4, m=1e6, one launch, the bench configuration): oracle parity on
    1024 seeded SNPs plus the first and last SNP of every int8 conversion chunk, every wave of
    128-column tiles, every 8192-column block, and the ragged tail; the FP64 DMMA path on the same
    sample plus its own panel-wave edges; then the planted-beta identity on ALL 1e6 SNPs."""
    cfg = gen.CONFIGS[2]
    P, L = n1e4_factor
    Xd = torch.empty((cfg.cols, cfg.n), dtype=torch.float64, device="cuda")
    for c in range(0, cfg.cols, 65536):
        k = min(65536, cfg.cols - c)
        glsmod.gen_xr_device(SEED, cfg.n, c, k, Xd[c:c + k])
    b, st, _ = run_gpu(glsmod, P, Xd, cfg.m, cfg.pR)
    assert np.all(st == 0)
    wave = 148 * 128                     # SNPs per wave of int8 tiles (pR = 1)
    edges = edge_set(cfg.m, wave, 8192, first_chunks=int8_chunk_bounds(cfg.m, wave))
    edges64 = edge_set(cfg.m, 148 * 64)  # FP64 path: 64-column panels, one per SM per wave
    rng = np.random.default_rng(2)
    sel = np.unique(np.concatenate([rng.choice(cfg.m, 1024, replace=False), edges, edges64]))
    XRs = np.concatenate([gen.make_XR(SEED, cfg.n, int(i), 1) for i in sel])
    b_or, st_or = oracle.gls_sequence(L, P.XL, P.y, XRs, 1, sel=sel, xr_is_selected=True)
    assert_parity(b[sel], st[sel], b_or, st_or, label="config2 sample")
    record_parity("config2 n=1e4 p=4 m=1e6: 1024 seeded + %d edge SNPs" % (len(sel) - 1024), b[sel], b_or, st_or)
    b64, st64, _ = run_gpu(glsmod, P, Xd, cfg.m, cfg.pR, path=glsmod.GLS_PATH_FP64)
    assert_parity(b64[sel], st64[sel], b_or, st_or, label="config2 sample, FP64 path")
    record_parity("config2, FP64 DMMA path: same %d SNPs" % len(sel), b64[sel], b_or, st_or)
    del b64, st64
    P0 = gen.config_problem(cfg, noise=0.0)
    b0, st0, _ = run_gpu(glsmod, P0, Xd, cfg.m, cfg.pR)
    ref = np.concatenate([P0.beta_L, [0.0]])
    assert np.all(st0 == 0)
    assert np.max(np.abs(b0 - ref)) / np.max(np.abs(P0.beta_L)) <= 1e-10


def test_config3_shape_sampled_parity(glsmod, n1e4_factor):
    """Config-3 shape (n=1e4, pL=16 covariates, pR=4, p=20) on 4000 groups: sampled oracle parity;
    the planted-beta identity on all groups."""
    cfg = gen.CONFIGS[3]
    m = 4000
    P = gen.config_problem(cfg)
    assert np.array_equal(P.M, n1e4_factor[0].M)  # configs 2-4 share M (same seed and n)
    L = n1e4_factor[1]
    XR = gen.make_XR(SEED, cfg.n, 0, m * cfg.pR)
    b, st, _ = run_gpu(glsmod, P, dev(XR), m, cfg.pR)
    sel = np.unique(np.concatenate([np.random.default_rng(3).choice(m, 24, replace=False), [0, 7, 8, 15, m - 1]]))
    b_or, st_or = oracle.gls_sequence(L, P.XL, P.y, XR, cfg.pR, sel=sel)
    assert_parity(b[sel], st[sel], b_or, st_or, label="config3 sample")
    record_parity("config3 shape (4000 groups): %d groups" % len(sel), b[sel], b_or, st_or)
    P0 = gen.config_problem(cfg, noise=0.0)
    b0, st0, _ = run_gpu(glsmod, P0, dev(XR), m, cfg.pR)
    ref = np.concatenate([P0.beta_L, np.zeros(cfg.pR)])
    assert np.max(np.abs(b0 - ref)) / np.max(np.abs(P0.beta_L)) <= 1e-10


def test_api_async_streams_and_errors(glsmod):
    """gls_solve_block_ex async mode + gls_sync, gls_set_stream onto a torch stream, status NULL,
    host b_out from device X_R, and argument errors (GLS_ERR_DIM / GLS_ERR_ARG)."""
    n, m = 256, 300
    P = gen.make_problem(n, 3, 1, seed=9)
    XR = gen.make_XR(9, n, 0, m)
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, 1)
    Xd = dev(XR)
    with glsmod.Context(n, 3, 1, dev(P.M), dev(P.XL), dev(P.y)) as ctx:
        s = torch.cuda.Stream()
        ctx.set_stream(s.cuda_stream)
        b1 = torch.empty((m, 4), dtype=torch.float64, device="cuda")
        ctx.solve_block(Xd, m, b1, None, async_=True)
        ctx.sync()
        assert_parity(b1.cpu().numpy(), np.zeros(m, np.int32), b_or, st_or, label="async")
        ctx.set_stream(None)
        bh = np.empty((m, 4))
        sh = np.empty(m, dtype=np.int32)
        ctx.solve_block(Xd, m, bh, sh)             # device X_R, host outputs
        np.testing.assert_array_equal(bh, b1.cpu().numpy())
        assert np.all(sh == 0)
        # async host stream: several calls in flight, one sync
        XRh = torch.from_numpy(XR).pin_memory()
        bh2 = torch.empty((m, 4), dtype=torch.float64).pin_memory()
        ctx.set_block_cols(64)
        ctx.solve_block(XRh[:100], 100, bh2[:100], None, async_=True)
        ctx.solve_block(XRh[100:], m - 100, bh2[100:], None, async_=True)
        ctx.sync()
        np.testing.assert_array_equal(bh2.numpy(), bh)
        with pytest.raises(glsmod.GLSError) as e:
            ctx.solve_block(Xd, 0, b1)
        assert e.value.code == 2
        import ctypes
        L = glsmod.load()
        assert L.gls_solve_block(ctx._h, None, m, b1.data_ptr()) == 1
        assert L.gls_solve_block_ex(ctx._h, Xd.data_ptr(), m, b1.data_ptr(), None, 7) == 1


@pytest.mark.parametrize("n", [1024, 1100, 3000])
def test_host_M_upload_overlapped_bitwise(glsmod, n):
    """M in (pinned or pageable) host memory reaches the device in 512-column chunks while the
    factorisation runs, each kernel waiting for the chunks it touches; the NotSPD tolerance comes
    from the host.  Results must equal those of a device-resident M bit for bit, and a NotSPD pivot
    in a late chunk must still be reported exactly."""
    pL, pR, m = 3, 1, 500
    P = gen.make_problem(n, pL, pR, seed=47)
    XR = gen.make_XR(47, n, 0, m)
    Xd = dev(XR)
    b_dev, st_dev, _ = run_gpu(glsmod, P, Xd, m, pR)
    for Mh in (torch.from_numpy(P.M).pin_memory(), np.ascontiguousarray(P.M)):
        with glsmod.Context(n, pL, pR, Mh, dev(P.XL), dev(P.y)) as ctx:
            b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
            ctx.solve_block(Xd, m, b)
            np.testing.assert_array_equal(b.cpu().numpy(), b_dev)
    M2 = P.M.copy()
    M2[n - 7, n - 7] = -1.0
    with pytest.raises(glsmod.GLSError) as eg:
        glsmod.Context(n, pL, pR, torch.from_numpy(M2).pin_memory(), dev(P.XL), dev(P.y))
    assert eg.value.code == 3


def test_repeated_create_destroy_is_deterministic(glsmod):
    """Pool-allocated contexts: create/solve/destroy three times gives identical bits."""
    n, m = 300, 150
    P = gen.make_problem(n, 2, 2, with_sex=False, seed=10)
    Xd = dev(gen.make_XR(10, n, 0, 2 * m))
    outs = []
    for _ in range(3):
        b, st, _ = run_gpu(glsmod, P, Xd, m, 2)
        outs.append(b)
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])


def test_cached_streams_across_overlapping_contexts(glsmod):
    """Contexts take their CUDA streams and events from a per-device cache and give them back on
    destroy.  A rolling window of three live contexts -- async solves still in flight when an older
    context is destroyed and a new one takes its streams, async creates from pinned host M, a user
    stream, timing and stream-report events -- must give every context exactly the bits of a context
    used alone."""
    cases = []
    for n, pL, pR, m, seed in ((1100, 3, 1, 700, 71), (1500, 2, 2, 300, 72)):
        P = gen.make_problem(n, pL, pR, seed=seed)
        XR = gen.make_XR(seed, n, 0, m * pR)
        b_ref, _, _ = run_gpu(glsmod, P, dev(XR), m, pR)
        cases.append((P, pR, m, dev(XR), torch.from_numpy(XR).to(torch.int8).pin_memory(), b_ref))
    user = torch.cuda.Stream()
    live = []

    def finish(entry):
        ctx, b, b_ref = entry
        ctx.sync()
        np.testing.assert_array_equal(b.cpu().numpy() if b.is_cuda else b.numpy(), b_ref)
        ctx.close()

    for it in range(12):
        P, pR, m, Xd, G8, b_ref = cases[it % 2]
        if it % 3 == 1:   # async create from pinned host buffers, then the host int8 stream
            ctx = glsmod.Context(P.n, P.pL, pR, torch.from_numpy(P.M).pin_memory(),
                                 torch.from_numpy(np.ascontiguousarray(P.XL)).pin_memory(),
                                 torch.from_numpy(P.y).pin_memory(), async_create=True)
            ctx.set_stream_report(True)
            b = torch.empty((m, P.pL + pR), dtype=torch.float64, pin_memory=True)
            ctx.solve_block_i8(G8, m, b, None, async_=True)
        else:             # device buffers, async solve, every other one on a user stream
            ctx = glsmod.Context(P.n, P.pL, pR, dev(P.M), dev(P.XL), dev(P.y))
            if it % 2 == 0:
                ctx.set_stream(user.cuda_stream)
            ctx.set_timing(True)
            b = torch.empty((m, P.pL + pR), dtype=torch.float64, device="cuda")
            ctx.solve_block(Xd, m, b, None, async_=True)
        live.append((ctx, b, b_ref))
        if len(live) == 3:
            finish(live.pop(0))   # destroyed while the two younger contexts still have work queued
    for entry in live:
        finish(entry)


def test_int8_genotype_entry_matches_double_entry(glsmod):
    """gls_solve_block_i8 (genotype codes) gives the same bits as gls_solve_block on the same
    values: device in place (ldg % 16 == 0), device with an odd leading dimension (staged),
    pinned and pageable host sources, host outputs; ragged n (not a multiple of 16 or 32)."""
    n, pL, pR, m = 1001, 3, 2, 333
    P = gen.make_problem(n, pL, pR, seed=23)
    XR = gen.make_XR(23, n, 0, m * pR)
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
    G = XR.astype(np.int8)
    with glsmod.Context(n, pL, pR, dev(P.M), dev(P.XL), dev(P.y)) as ctx:
        ref = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
        ctx.solve_block(dev(XR), m, ref)
        ref = ref.cpu().numpy()
        assert_parity(ref, np.zeros(m, np.int32), b_or, st_or, label="i8 ref")
        for ldg in (1008, 1001, 1013):
            Gp = np.zeros((m * pR, ldg), dtype=np.int8)
            Gp[:, :n] = G
            Gd = torch.from_numpy(Gp).cuda()
            b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
            st = torch.empty(m, dtype=torch.int32, device="cuda")
            ctx.solve_block_i8(Gd, m, b, st, ldg=ldg)
            np.testing.assert_array_equal(b.cpu().numpy(), ref)
            assert int(st.sum()) == 0
            bh = np.empty((m, pL + pR))
            ctx.set_block_cols(2 * 64)
            ctx.solve_block_i8(torch.from_numpy(Gp).pin_memory(), m, bh, ldg=ldg)
            np.testing.assert_array_equal(bh, ref)
            bh2 = np.empty((m, pL + pR))
            ctx.solve_block_i8(Gp, m, bh2, ldg=ldg)
            np.testing.assert_array_equal(bh2, ref)
        with pytest.raises(glsmod.GLSError) as e:
            ctx.solve_block_i8(torch.from_numpy(G).cuda(), m, torch.empty((m, 5), dtype=torch.float64,
                                                                           device="cuda"), ldg=n - 1)
        assert e.value.code == 1


def test_timing_hooks_and_counts(glsmod):
    n, m = 512, 4000
    P = gen.make_problem(n, 3, 1, seed=24)
    Xd = dev(gen.make_XR(24, n, 0, m))
    with glsmod.Context(n, 3, 1, dev(P.M), dev(P.XL), dev(P.y)) as ctx:
        ctx.set_timing(True)
        b = torch.empty((m, 4), dtype=torch.float64, device="cuda")
        ctx.solve_block(Xd, m, b)
        t = ctx.read_timing()
        # timed launches: the conversion, the int8 kernel, and the block's two (gated, idle) FP64
        # fallback launches -- compacted and in place (reading A16)
        assert t["launches"] == 4 and t["int8_ms"] > 0 and t["conv_ms"] > 0, t
        assert ctx.path_counts() == (1, 0)
        ctx.set_path(glsmod.GLS_PATH_FP64)
        ctx.solve_block(Xd, m, b)
        t = ctx.read_timing()
        assert t["launches"] == 1 and t["fp64_ms"] > 0 and t["int8_ms"] == 0, t
        assert ctx.path_counts() == (1, 1)


def test_solve_file_sync_and_async_bitwise(glsmod, tmp_path):
    """Out-of-core from secondary storage (§4): Alg. 7 (sync) and Alg. 8 (double-buffered) over FP64
    and int8-code X_R files, with a warm-up block (§4.3), give exactly the in-core bits; the report
    accounts for every block and byte; bad files are GLS_ERR_ARG."""
    n, pL, pR, m = 700, 3, 1, 3000
    P = gen.make_problem(n, pL, pR, seed=25)
    XR = gen.make_XR(25, n, 0, m)
    hdr = np.arange(8, dtype=np.float64)  # 64-byte header before the stream
    f64 = tmp_path / "xr_f64.bin"
    with open(f64, "wb") as f:
        f.write(hdr.tobytes())
        f.write(XR.tobytes())
    i8 = tmp_path / "xr_i8.bin"
    XR.astype(np.int8).tofile(i8)
    bpath, spath = str(tmp_path / "b.bin"), str(tmp_path / "st.bin")
    with glsmod.Context(n, pL, pR, dev(P.M), dev(P.XL), dev(P.y)) as ctx:
        ref = torch.empty((m, 4), dtype=torch.float64, device="cuda")
        ctx.solve_block(dev(XR), m, ref)
        ref = ref.cpu().numpy()
        b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR[:200], pR)
        assert_parity(ref[:200], np.zeros(200, np.int32), b_or, st_or, label="file ref")
        for mode in (glsmod.GLS_OOC_SYNC, glsmod.GLS_OOC_ASYNC):
            for path, elem, off in ((str(f64), 8, 64), (str(i8), 1, 0)):
                rep = ctx.solve_file(path, m, bpath, spath, elem_bytes=elem, xr_offset=off, block_groups=700,
                                     warmup_groups=100, mode=mode)
                b = np.fromfile(bpath).reshape(m, 4)
                st = np.fromfile(spath, dtype=np.int32)
                np.testing.assert_array_equal(b, ref)
                assert st.shape == (m,) and not st.any()
                assert rep["blocks"] == 1 + (m - 100 + 699) // 700
                assert rep["bytes_read"] == m * n * elem and rep["bytes_written"] == m * 4 * 8
                assert rep["wall_s"] >= rep["compute_s"] > 0 and rep["read_wait_s"] >= rep["first_load_s"] >= 0
        with pytest.raises(glsmod.GLSError) as e:
            ctx.solve_file(str(tmp_path / "missing.bin"), m, bpath)
        assert e.value.code == 1
        # a b file whose writes fail (ENOSPC): both modes must report the failure, never GLS_OK
        if os.path.exists("/dev/full"):
            for mode in (glsmod.GLS_OOC_SYNC, glsmod.GLS_OOC_ASYNC):
                with pytest.raises(glsmod.GLSError) as e:
                    ctx.solve_file(str(f64), m, "/dev/full", elem_bytes=8, xr_offset=64, block_groups=300,
                                   mode=mode)
                assert e.value.code == 1
        short = tmp_path / "short.bin"
        XR[: m // 2].tofile(short)
        for mode in (glsmod.GLS_OOC_SYNC, glsmod.GLS_OOC_ASYNC):
            with pytest.raises(glsmod.GLSError) as e:
                ctx.solve_file(str(short), m, bpath, block_groups=500, mode=mode)
            assert e.value.code == 1


def test_algorithm_ladder_agrees(glsmod):
    """NEXT-2: seq-gls (Alg. 4: every problem's p columns whitened, FP64 path) and black-box (Alg. 3: a
    factorization per problem) on the B200 kernels reproduce hp-gwas's b -- an
    independent GPU-side check of the Fig. 1 partition."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "ladder", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "ladder.py"))
    ladder = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ladder)
    n, pL, pR, m, m_bb, seed = 300, 3, 1, 300, 6, 26
    out = ladder.run(n, pL, pR, m, m_bb, seed=seed, return_b=True)
    # every rung against the oracle on the same seeded problem (ladder.run draws it the same way)
    P = gen.make_problem(n, pL, pR, with_sex=True, seed=seed)
    XR = gen.make_XR(seed, n, 0, m * pR)
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
    for rung, b in out["_b"].items():
        k = len(b)
        assert_parity(b, np.zeros(k, np.int32), b_or[:k], st_or[:k], label="ladder " + rung)
        record_parity("ladder n=300 p=4: %s (%d problems)" % (rung, k), b, b_or[:k])


def test_config3_full_size_sampled_parity(glsmod, n1e4_factor):
    """Config 3 at full size (n=1e4, pL=16, pR=4, 5e5 groups = 2e6 columns, 160 GB of X_R in HBM; the
    bench launch): oracle parity on 512 seeded groups plus the first and last group of every
    128-column tile pair at the start and end, of every wave and of every int8 conversion chunk, and
    the planted-beta identity on every group."""
    cfg = gen.CONFIGS[3]
    torch.cuda.empty_cache()  # earlier tests' X_R buffers sit in torch's cache
    glsmod.release_cached_memory()  # and earlier contexts' buffers in the library's pool
    free, _ = torch.cuda.mem_get_info()
    if free < 175e9:
        pytest.skip("needs ~170 GB of free device memory")
    P = gen.config_problem(cfg)
    assert np.array_equal(P.M, n1e4_factor[0].M)
    Lf = n1e4_factor[1]
    cols = cfg.m * cfg.pR
    Xd = torch.empty((cols, cfg.n), dtype=torch.float64, device="cuda")
    for c in range(0, cols, 65536):
        k = min(65536, cols - c)
        glsmod.gen_xr_device(SEED, cfg.n, c, k, Xd[c:c + k])
    b, st, _ = run_gpu(glsmod, P, Xd, cfg.m, cfg.pR)
    assert np.all(st == 0)
    tile_g = 32  # groups per 128-column tile at pR = 4; a CTA pair covers 2 tiles
    wave_g = 148 * tile_g
    head_tail = [x for t in range(4) for x in (t * tile_g, (t + 1) * tile_g - 1)]
    head_tail += [cfg.m - 1 - x for x in head_tail]
    edges = edge_set(cfg.m, wave_g, first_chunks=int8_chunk_bounds(cfg.m, wave_g))
    sel = np.unique(np.concatenate([np.random.default_rng(4).choice(cfg.m, 512, replace=False), edges,
                                    head_tail, [7, 8]]))
    XRs = np.concatenate([gen.make_XR(SEED, cfg.n, int(i) * cfg.pR, cfg.pR) for i in sel])
    b_or, st_or = oracle.gls_sequence(Lf, P.XL, P.y, XRs, cfg.pR, sel=sel, xr_is_selected=True)
    assert_parity(b[sel], st[sel], b_or, st_or, label="config3 full sample")
    record_parity("config3 n=1e4 p=20 m=5e5: 512 seeded + %d edge groups" % (len(sel) - 512), b[sel], b_or, st_or)
    P0 = gen.config_problem(cfg, noise=0.0)
    b0, st0, _ = run_gpu(glsmod, P0, Xd, cfg.m, cfg.pR)
    del Xd
    ref = np.concatenate([P0.beta_L, np.zeros(cfg.pR)])
    assert np.all(st0 == 0)
    assert np.max(np.abs(b0 - ref)) / np.max(np.abs(P0.beta_L)) <= 1e-10


def test_config4_full_stream(glsmod, n1e4_factor):
    """Config 4 in the bench launch configuration (bench.py run_ooc): m = 1e7 SNPs streamed from
    pinned host memory as int8 genotype codes through the double-buffered H2D pipeline (Alg. 8), the
    host blocks cycled from a pool of 4 distinct blocks (block j = pool block j mod 4).
      * every one of the 1e7 b rows equals, bit for bit, the in-HBM solve of its pool block's SNP;
      * 2e6 SNPs of the same stream from FP64 host X_R (a pool of 2 blocks) equal it bit for bit;
      * the oracle checks 1024 seeded SNPs of the distinct region plus the first and last SNP of
        every host block, wave of tiles and 8192-column block in it."""
    from paper_1210_7325_b200 import ooc
    cfg = gen.CONFIGS[4]
    P, Lf = n1e4_factor
    n, m = cfg.n, cfg.m
    blk = ooc.host_block_groups(torch.cuda.get_device_properties(0).multi_processor_count, cfg.pR)
    PB = 4
    distinct = PB * blk
    Xd = torch.empty((distinct, n), dtype=torch.float64, device="cuda")
    for c in range(0, distinct, 65536):
        k = min(65536, distinct - c)
        glsmod.gen_xr_device(SEED, n, c, k, Xd[c:c + k])
    pool8 = torch.empty((PB, blk, n), dtype=torch.int8).pin_memory()
    for k in range(PB):
        pool8[k].copy_(Xd[k * blk:(k + 1) * blk].to(torch.int8))
    with glsmod.Context(n, cfg.pL, cfg.pR, dev(P.M), dev(P.XL), dev(P.y)) as ctx:
        bd = torch.empty((distinct, 4), dtype=torch.float64, device="cuda")
        ctx.solve_block(Xd, distinct, bd)
        bd = bd.cpu()
        b = torch.empty((m, 4), dtype=torch.float64).pin_memory()
        st = torch.empty(m, dtype=torch.int32).pin_memory()
        nblk = ooc.stream_from_pool(ctx, pool8, m, blk, b, st, codes=True)
        assert nblk == (m + blk - 1) // blk
        assert not st.numpy().any()
        for j in range(nblk):
            lo, cnt = j * blk, min(blk, m - j * blk)
            k = j % PB
            assert torch.equal(b[lo:lo + cnt], bd[k * blk:k * blk + cnt]), "stream block %d" % j
        # FP64 host X_R through the same pipeline (8 bytes per genotype over PCIe)
        del pool8
        m64 = 2_000_000
        pool64 = torch.empty((2, blk, n), dtype=torch.float64).pin_memory()
        for k in range(2):
            pool64[k].copy_(Xd[k * blk:(k + 1) * blk])
        b64 = torch.empty((m64, 4), dtype=torch.float64).pin_memory()
        st64 = torch.empty(m64, dtype=torch.int32).pin_memory()
        nb64 = ooc.stream_from_pool(ctx, pool64, m64, blk, b64, st64, codes=False)
        for j in range(nb64):
            lo, cnt = j * blk, min(blk, m64 - j * blk)
            k = j % 2
            assert torch.equal(b64[lo:lo + cnt], bd[k * blk:k * blk + cnt]), "FP64 stream block %d" % j
        del pool64
    del Xd
    bd = bd.numpy()
    wave = 148 * 128
    sel = np.unique(np.concatenate([np.random.default_rng(44).choice(distinct, 1024, replace=False),
                                    edge_set(distinct, blk, wave, 8192)]))
    XRs = np.concatenate([gen.make_XR(SEED, n, int(i), 1) for i in sel])
    b_or, st_or = oracle.gls_sequence(Lf, P.XL, P.y, XRs, 1, sel=sel, xr_is_selected=True)
    assert_parity(bd[sel], np.zeros(len(sel), np.int32), b_or, st_or, label="config4 sample")
    record_parity("config4 n=1e4 p=4 m=1e7 streamed: 1024 seeded + %d edge SNPs" % (len(sel) - 1024),
                  bd[sel], b_or, st_or)


@pytest.mark.parametrize("n,pL,pR,m", [(500, 3, 1, 300), (260, 16, 4, 40), (300, 0, 2, 50)])
def test_gwfgls_rung_matches_oracle(glsmod, n, pL, pR, m):
    """NEXT-2: GenABEL's gwfgls (Alg. 6) on the B200 kernels -- explicit M^-1, per-column
    gemv (as listed) or one GEMM per block, full p x p S_i = W^T X_i, gesv -- reaches Eq. (1)'s b: every
    problem against the oracle in both modes; a zero SNP is RankDeficient (NaN, status 1)."""
    P = gen.make_problem(n, pL, pR, with_sex=pL >= 3, seed=28 + n)
    XR = gen.make_XR(28 + n, n, 0, m * pR)
    XR[3 * pR:4 * pR] = 0.0  # problem 3: an all-zero genotype block
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
    assert st_or[3] == 1
    with glsmod.Gwfgls(n, pL, pR, dev(P.M), dev(P.XL) if pL else None, dev(P.y)) as g:
        for mode in (glsmod.GLS_GWFGLS_GEMV, glsmod.GLS_GWFGLS_GEMM):
            b = torch.empty((m, pL + pR), dtype=torch.float64, device="cuda")
            st = torch.empty(m, dtype=torch.int32, device="cuda")
            g.solve(dev(XR), m, b, st, mode=mode)
            b, st = b.cpu().numpy(), st.cpu().numpy()
            assert_parity(b, st, b_or, st_or, label="gwfgls mode %d" % mode)
        assert g.kernel_launches > 0
        with pytest.raises(glsmod.GLSError):
            g.solve(dev(XR), 0, torch.empty((1, pL + pR), dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("n", [1100, 4100])
def test_create_async_bitwise(glsmod, n):
    """gls_create_async (Alg. 8 lines 1-5 overlapped with the first block's H2D): the same shared state
    and the same b bit for bit as gls_create, with M / X_L / y pinned on the host and a host X_R block
    (codes and FP64) streamed while the factorisation may still run; and against the oracle."""
    from paper_1210_7325_b200 import multi
    pL, pR, m = 3, 1, 700
    P = gen.make_problem(n, pL, pR, seed=61)
    XR = gen.make_XR(61, n, 0, m)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    Mh, XLh, yh = pin(P.M), pin(P.XL), pin(P.y)
    G = pin(XR.astype(np.int8))
    Xh = pin(XR)
    with glsmod.Context(n, pL, pR, Mh, XLh, yh) as ref:
        dig_ref = multi.shared_state_digest(ref)
        b_ref = torch.empty((m, pL + pR), dtype=torch.float64, pin_memory=True)
        ref.solve_block_i8(G, m, b_ref)
        b_ref64 = torch.empty((m, pL + pR), dtype=torch.float64, pin_memory=True)
        ref.solve_block(Xh, m, b_ref64)
    for entry in ("i8", "f64", "sync"):
        with glsmod.Context(n, pL, pR, Mh, XLh, yh, async_create=True) as ctx:
            b = torch.empty((m, pL + pR), dtype=torch.float64, pin_memory=True)
            st = torch.empty(m, dtype=torch.int32, pin_memory=True)
            if entry == "i8":
                ctx.solve_block_i8(G, m, b, st)         # synchronous: resolves the create at its end
            elif entry == "f64":
                ctx.solve_block(Xh, m, b, st, async_=True)
                ctx.sync()
            else:
                ctx.sync()
                ctx.solve_block(Xh, m, b, st)
            np.testing.assert_array_equal(b.numpy(), (b_ref if entry == "i8" else b_ref64).numpy())
            assert multi.shared_state_digest(ctx) == dig_ref
    b_or, st_or = oracle.solve(P.M, P.XL, P.y, XR, pR)
    assert_parity(b_ref.numpy(), st.numpy(), b_or, st_or, label="create_async n=%d" % n)


def test_create_async_not_spd(glsmod):
    """A non-SPD M under gls_create_async: the create returns OK, the first synchronising call reports
    GLS_ERR_NOT_SPD with the oracle's pivot, the context is failed afterwards, destroy is clean."""
    import ctypes
    n, piv = 1100, 777
    P = gen.make_problem(n, 3, 1, seed=62)
    M = P.M.copy()
    M[piv, piv] = -1.0
    with pytest.raises(oracle.NotSPD) as ei:
        oracle.cholesky(M)
    assert ei.value.pivot == piv
    L = glsmod.load()
    Mh = torch.from_numpy(M).pin_memory()
    XLd, yd = dev(P.XL), dev(P.y)
    G = torch.from_numpy(gen.make_XR(62, n, 0, 50).astype(np.int8)).pin_memory()
    b = torch.empty((50, 4), dtype=torch.float64, pin_memory=True)
    h = ctypes.c_void_p()
    assert L.gls_create_async(n, 3, 1, Mh.data_ptr(), XLd.data_ptr(), yd.data_ptr(), ctypes.byref(h)) == 0
    assert L.gls_solve_block_i8(h, G.data_ptr(), n, 50, b.data_ptr(), None, 1) == 0   # enqueued
    assert L.gls_sync(h) == 3                                                          # GLS_ERR_NOT_SPD
    assert L.gls_failed_pivot(h) == piv
    assert L.gls_sync(h) == 0 and L.gls_solve_block_i8(h, G.data_ptr(), n, 50, b.data_ptr(), None, 0) == 6
    L.gls_destroy(h)
    # the same through the binding: the synchronous solve raises, with the pivot on the context
    with glsmod.Context(n, 3, 1, Mh, XLd, yd, async_create=True) as ctx:
        with pytest.raises(glsmod.GLSError) as eg:
            ctx.solve_block_i8(G, 50, b)
        assert eg.value.code == 3 and ctx.failed_pivot == piv


def test_create_bitwise_independent_of_schedule(glsmod):
    """The create's shared state (T digits, packed T, aux, V digits, G) is bit-for-bit the same under
    every scheduling switch of the factorisation: TMA GEMM tile order (cost-ordered snake vs
    round-robin), look-ahead products after vs beside the main stream, the free-SM budget of the
    off-critical-path products -- no result depends on which CTA or stream ran a tile first.  Each
    setting runs in its own process (the switches are read once per process)."""
    import json, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, json, numpy as np, torch; sys.path.insert(0, %r); import gen; "
            "import paper_1210_7325_b200 as pkg; from paper_1210_7325_b200 import multi; out = {}\n"
            "for n in (1500, 4097):\n"
            "    P = gen.make_problem(n, 3, 1)\n"
            "    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()\n"
            "    with pkg.Context(n, 3, 1, d(P.M), d(P.XL), d(P.y)) as c: out[n] = multi.shared_state_digest(c)\n"
            "print(json.dumps(out))" % root)
    runs = {}
    for name, env in [("default", {}), ("round_robin", {"GLS_DGEMM_SCHED": "0"}),
                      ("side_concurrent", {"GLS_SIDE_AFTER": "0"}), ("free48", {"GLS_CHOL_FREE_SMS": "48"})]:
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        runs[name] = json.loads(r.stdout.strip().splitlines()[-1])
    for name, dg in runs.items():
        assert dg == runs["default"], name


def test_hot_kernels_bitwise_under_perturbation(glsmod):
    """Race evidence without a race detector (compute-sanitizer is closed on this pool): the int8
    tcgen05 kernel (mbarrier rings, TMEM hand-over between the MMA issuer and the epilogue, the CTA
    pair's remote arrivals, the convert-ahead warps) and the FP64 DMMA kernel give the same bits when
    their timing is perturbed -- fewer CTA pairs / CTAs (another tile schedule), in-kernel clock
    counters on (GLS_OZ_PROF), and a concurrent GEMM load on another stream competing for the SMs.
    A missing wait or a premature release would show up as a changed bit in some run."""
    import json, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # n >= 4096 so the convert-ahead warps run; 3 chunks of tiles plus a ragged tail
    code = ("import sys, hashlib, numpy as np, torch; sys.path.insert(0, %r); import gen; "
            "import paper_1210_7325_b200 as pkg\n"
            "n, m = 4100, 3 * 18944 + 77\n"
            "P = gen.make_problem(n, 3, 1, seed=71)\n"
            "d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()\n"
            "X = torch.empty((m, n), dtype=torch.float64, device='cuda')\n"
            "pkg.gen_xr_device(71, n, 0, m, X)\n"
            "load = sys.argv[1] == 'load'\n"
            "if load:\n"
            "    s2 = torch.cuda.Stream(); a = torch.randn(8192, 8192, device='cuda')\n"
            "out = []\n"
            "with pkg.Context(n, 3, 1, d(P.M), d(P.XL), d(P.y)) as c:\n"
            "    for path in (pkg.GLS_PATH_AUTO, pkg.GLS_PATH_FP64):\n"
            "        c.set_path(path)\n"
            "        b = torch.empty((m, 4), dtype=torch.float64, device='cuda')\n"
            "        if load:\n"
            "            with torch.cuda.stream(s2):\n"
            "                for _ in range(30): a = a @ a; a /= a.abs().max()\n"
            "        c.solve_block(X, m, b)\n"
            "        out.append(hashlib.sha256(b.cpu().numpy().tobytes()).hexdigest())\n"
            "print(' '.join(out))" % root)
    runs = {}
    for name, env, arg in [("default", {}, "-"), ("pairs7", {"GLS_OZ_PAIRS": "7", "GLS_FP64_CTAS": "13"}, "-"),
                           ("prof", {"GLS_OZ_PROF": "1"}, "-"), ("load", {}, "load"),
                           ("pairs33_load", {"GLS_OZ_PAIRS": "33", "GLS_FP64_CTAS": "61"}, "load")]:
        r = subprocess.run([sys.executable, "-c", code, arg], env={**os.environ, **env}, capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, (name, r.stderr[-2000:])
        runs[name] = r.stdout.strip().splitlines()[-1].split()
    for name, h in runs.items():
        assert h == runs["default"], (name, h, runs["default"])


def test_large_n_planted_beta(glsmod):
    """Maximum-size check far above the configs: n = 49 999 (odd, so every tile, chunk and 16-byte
    pitch is ragged; 1563 row blocks of the int8 digit tiles, int32 digit sums up to 127 * 2 * n),
    noise-free y = X_L beta.  No oracle can factor this M in a test's time, so the pin is the
    planted-beta identity b_i = (beta, 0) (PAPER.md:28-39 with y in span(X_L)), on both arithmetic
    paths: the int8 tcgen05 path on three chunks of SNPs plus a ragged tail, the FP64 DMMA path on a
    subset."""
    import gc
    gc.collect()
    torch.cuda.empty_cache()          # earlier tests' cached blocks (config 3 held 160 GB)
    glsmod.release_cached_memory()
    n, pL, pR = 49_999, 3, 1
    m = 2 * 18944 + 333
    P = gen.make_problem(n, pL, pR, seed=81, noise=0.0)
    Xd = torch.empty((m * pR, n), dtype=torch.float64, device="cuda")
    glsmod.gen_xr_device(81, n, 0, m * pR, Xd)
    ref = np.concatenate([P.beta_L, [0.0]])
    scale = np.max(np.abs(P.beta_L))
    with glsmod.Context(n, pL, pR, dev(P.M), dev(P.XL), dev(P.y)) as ctx:
        for path, mm in ((glsmod.GLS_PATH_AUTO, m), (glsmod.GLS_PATH_FP64, 2000)):
            ctx.set_path(path)
            b = torch.empty((mm, pL + pR), dtype=torch.float64, device="cuda")
            st = torch.empty(mm, dtype=torch.int32, device="cuda")
            ctx.solve_block(Xd, mm, b, st)
            counts = ctx.path_counts()
            b, st = b.cpu().numpy(), st.cpu().numpy()
            assert np.all(st == 0)
            err = float(np.max(np.abs(b - ref)) / scale)
            assert err <= 1e-9, (path, err)
            if path == glsmod.GLS_PATH_AUTO:
                assert counts[0] > 0, counts  # the int8 kernel did the work


def test_strong_shards_bitwise_for_every_world_size(glsmod):
    """b bitwise independent of the number of GPUs.  The strong-scaling split of the bench
    (rank r of G owns problems [floor(r m / G), floor((r+1) m / G)), each rank with its own create --
    the redundant factorisation) is replayed on this GPU for G = 2, 4, 8: every
    shard's b, from its own context, equals the rows of the single-GPU run bit for bit (shard edges
    fall inside conversion chunks, waves and tiles)."""
    from paper_1210_7325_b200 import multi
    n, pL, pR = 10_000, 3, 1
    m = 3 * 18944 + 1234
    P = gen.make_problem(n, pL, pR, seed=91)
    Xd = torch.empty((m * pR, n), dtype=torch.float64, device="cuda")
    glsmod.gen_xr_device(91, n, 0, m * pR, Xd)
    b_full, st_full, _ = run_gpu(glsmod, P, Xd, m, pR)
    for G in (2, 4, 8):
        parts = []
        for r in range(G):
            lo, hi = multi.snp_range(m, G, r)
            b_r, _, _ = run_gpu(glsmod, P, Xd[lo * pR:hi * pR], hi - lo, pR)
            parts.append(b_r)
        np.testing.assert_array_equal(np.concatenate(parts), b_full, err_msg="G=%d" % G)
