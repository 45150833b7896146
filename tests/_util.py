"""Shared helpers for the parity tests (no method arithmetic here)."""
import numpy as np

# North-star tolerance: b_i matches the oracle within 1e-9 relative per entry, read as the
# guarded metric of DESIGN.md reading A10 (entries below 1e-3 * ||b_i||_inf are compared
# against that floor instead of their own near-zero magnitude).
PARITY_TOL = 1e-9


def guarded_rel_err(b_gpu: np.ndarray, b_ora: np.ndarray) -> float:
    b_gpu = np.asarray(b_gpu, dtype=np.float64)
    b_ora = np.asarray(b_ora, dtype=np.float64)
    assert b_gpu.shape == b_ora.shape
    if b_ora.size == 0:
        return 0.0
    floor = 1e-3 * np.max(np.abs(b_ora), axis=1, keepdims=True)
    den = np.maximum(np.abs(b_ora), floor)
    den = np.where(den > 0, den, 1.0)
    return float(np.max(np.abs(b_gpu - b_ora) / den))


def normwise_err(b_gpu, b_ora) -> float:
    num = np.linalg.norm(np.asarray(b_gpu) - np.asarray(b_ora), axis=1)
    den = np.maximum(np.linalg.norm(np.asarray(b_ora), axis=1), 1e-300)
    return float(np.max(num / den)) if num.size else 0.0


def assert_parity(b_gpu, st_gpu, b_ora, st_ora, tol=PARITY_TOL, label=""):
    b_gpu = np.asarray(b_gpu)
    st_gpu = np.asarray(st_gpu)
    np.testing.assert_array_equal(st_gpu, st_ora, err_msg="status mismatch " + label)
    ok = st_ora == 0
    if np.any(~ok):
        assert np.all(np.isnan(b_gpu[~ok])), "RankDeficient rows must be NaN " + label
    err = guarded_rel_err(b_gpu[ok], np.asarray(b_ora)[ok])
    assert err <= tol, "guarded relative error %.3e > %.1e %s" % (err, tol, label)
    return err


# ----------------------------------------------------------------------------- parity report
# Every full-size parity test records (label, problems checked, max guarded error, max norm-wise
# error); conftest.py prints the table at the end of the session, also under -q.
PARITY_REPORT = []


def record_parity(label, b_gpu, b_ora, st_ora=None):
    b_gpu = np.asarray(b_gpu)
    b_ora = np.asarray(b_ora)
    ok = np.ones(len(b_ora), bool) if st_ora is None else (np.asarray(st_ora) == 0)
    g = guarded_rel_err(b_gpu[ok], b_ora[ok])
    nw = normwise_err(b_gpu[ok], b_ora[ok])
    PARITY_REPORT.append((label, int(len(b_ora)), g, nw))
    return g, nw


def edge_set(m, *periods, first_chunks=None):
    """Sorted problem indices at the edges of a launch: for every boundary B of every period
    (multiples of the period) and of the explicit chunk boundaries, the problems B - 1 and B; plus
    0 and m - 1 (the ragged tail)."""
    bnd = {0, m}
    for per in periods:
        bnd.update(range(0, m, per))
    if first_chunks is not None:
        bnd.update(first_chunks)
    out = set()
    for b in bnd:
        for i in (b - 1, b):
            if 0 <= i < m:
                out.add(i)
    return np.array(sorted(out), dtype=np.int64)


def int8_chunk_bounds(m_groups, wave_groups, ahead=True):
    """Chunk boundaries of one device block on the int8 path (gls_api.cu run_kernel): 1, 2, .., 8,
    8, .. waves with convert-ahead (n >= 4096), else chunks of 8 waves."""
    bnd = [0]
    j = 1
    while bnd[-1] < m_groups:
        bnd.append(min(m_groups, bnd[-1] + (min(j, 8) if ahead else 8) * wave_groups))
        j += 1
    return bnd
