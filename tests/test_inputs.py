"""Synthetic input generators (rig_inputs): canonical CSR, recipe shapes,
determinism.  CPU-only."""
import numpy as np
import pytest

from rig_inputs import make, make_small


def check_canonical(w):
    rp, ci, v = w.row_ptr, w.col_idx, w.val
    assert rp.dtype == np.int64 and ci.dtype == np.int32 and v.dtype == np.float64
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == ci.size == v.size
    assert ci.min() >= 0 and ci.max() < w.ncols
    d = np.diff(ci.astype(np.int64))
    starts = rp[1:-1][np.diff(rp)[1:] > 0]  # positions where a new nonempty row starts
    bad = d <= 0
    bad[starts[starts > 0] - 1] = False
    assert not bad.any(), "columns not strictly increasing within a row"
    assert np.all(v != 0) and np.all(np.isfinite(v))
    assert w.part.dtype == np.int32 and w.part.size == w.n
    assert w.part.min() >= 0 and w.part.max() < w.K


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6, 7])
def test_small_configs_canonical_and_deterministic(cfg):
    a, b = make_small(cfg), make_small(cfg)
    check_canonical(a)
    assert a.row_ptr.tobytes() == b.row_ptr.tobytes()
    assert a.col_idx.tobytes() == b.col_idx.tobytes()
    assert a.val.tobytes() == b.val.tobytes()
    assert a.part.tobytes() == b.part.tobytes()


def test_recipe_shapes():
    # f3 stress configs: mean row length ~12.3 (Zipf + 8), and 64-entry rows
    # with every column within 1000 of the diagonal
    w = make_small(6)
    assert 11.0 < w.nnz / w.n < 13.5
    w = make_small(7)
    assert np.all(np.diff(w.row_ptr) == 64)
    rows = np.repeat(np.arange(w.n), 64)
    assert np.abs(w.col_idx.astype(np.int64) - rows).max() <= 1000
    w = make(2)
    assert w.n == 1_000_000 and w.nnz == 4_996_000  # N^2 + 4N(N-1)
    w = make_small(3)
    N = 23
    assert w.nnz == N ** 3 + 6 * N * N * (N - 1)
    w = make_small(5)
    assert np.all(np.diff(w.row_ptr) == 23)
    rows = np.repeat(np.arange(w.n), 23)
    dist = np.abs(w.col_idx.astype(np.int64) - rows)
    per_row_far = np.bincount(rows[dist > 50], minlength=w.n)
    per_row_band = np.bincount(rows[(dist >= 1) & (dist <= 50)], minlength=w.n)
    assert np.all(per_row_far == 3) and np.all(per_row_band == 19)
    # diagonal dominance: a_ii = 1 + sum |a_ij|
    sample = np.arange(0, w.n, 997)
    dpos = w.row_ptr[sample] + np.array([np.searchsorted(w.col_idx[w.row_ptr[i]:w.row_ptr[i + 1]], i)
                                         for i in sample])
    assert np.all(w.val[dpos] > 1.0)
    w = make_small(4)
    lens = np.diff(w.row_ptr)
    assert lens.min() >= 1 and lens.max() <= 5000
    has_diag = np.zeros(w.n, bool)
    rows = np.repeat(np.arange(w.n), lens)
    has_diag[rows[w.col_idx == rows]] = True
    assert has_diag.all()
