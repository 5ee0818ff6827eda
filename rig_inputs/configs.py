"""Generators for the five BASELINE.json configurations (and reduced-size twins).

Recipes follow SURVEY.md §8(d) table D2, which restates BASELINE.json's
``configs`` as concrete synthetic inputs standing in for the paper's 76
SuiteSparse matrices (Table matrix_prop; not available here).

RNG: numpy PCG64 ``default_rng(171007769 + cfg_id)`` for matrices and
``default_rng(171007769 + 1000 + cfg_id)`` for partitions.  Every matrix is
emitted as canonical CSR (row_ptr int64[n+1], col_idx int32[nnz] strictly
increasing per row, val float64[nnz], no explicit zeros).

Nothing here computes any part of the method.
"""
from __future__ import annotations

import dataclasses

import numpy as np

SEED_BASE = 171007769

CONFIG_NAMES = {
    1: "tiny",
    2: "stencil2d",
    3: "stencil3d",
    4: "powerlaw",
    5: "banded",
    6: "powerlaw12",
    7: "denserows",
}


@dataclasses.dataclass
class Workload:
    name: str
    cfg_id: int
    n: int
    ncols: int
    row_ptr: np.ndarray  # int64[n+1]
    col_idx: np.ndarray  # int32[nnz]
    val: np.ndarray      # float64[nnz]
    scale_rows: int
    drop_tol: float
    part: np.ndarray     # int32[n]
    K: int
    recipe: str

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


# --------------------------------------------------------------------------
# CSR assembly helpers (pure data movement)
# --------------------------------------------------------------------------

def _rows_to_csr(n, cols2d, mask2d, vals2d):
    """Flatten fixed-width per-row candidate lists whose valid entries are
    already in ascending column order."""
    counts = mask2d.sum(axis=1).astype(np.int64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col = cols2d[mask2d].astype(np.int32)
    val = vals2d[mask2d].astype(np.float64)
    return row_ptr, col, val


def from_triplets(n, ncols, rows, cols, vals):
    """Canonical CSR from COO triplets (duplicates are an error)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    keep = vals != 0.0
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size > 1:
        dup = (rows[1:] == rows[:-1]) & (cols[1:] == cols[:-1])
        if dup.any():
            raise ValueError("duplicate (row, col) entries")
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return row_ptr, cols.astype(np.int32), vals


def from_dense(D):
    D = np.asarray(D, dtype=np.float64)
    r, c = np.nonzero(D)
    return from_triplets(D.shape[0], D.shape[1], r, c, D[r, c])


def _nonzero_normal(rng, size):
    v = rng.standard_normal(size)
    while True:
        z = v == 0.0
        if not z.any():
            return v
        v[z] = rng.standard_normal(int(z.sum()))


def _nonzero_uniform(rng, lo, hi, size):
    v = rng.uniform(lo, hi, size)
    while True:
        z = v == 0.0
        if not z.any():
            return v
        v[z] = rng.uniform(lo, hi, int(z.sum()))


# --------------------------------------------------------------------------
# Partitions (last column; SPEC.md:262-270 sizing)
# --------------------------------------------------------------------------

def part_contiguous(n, K):
    """Uniform contiguous block-row partition (the paper's UP):
    part sizes differ by at most one, larger parts first (n=10,K=3 -> 4,3,3)."""
    base, extra = divmod(n, K)
    sizes = np.full(K, base, dtype=np.int64)
    sizes[:extra] += 1
    return np.repeat(np.arange(K, dtype=np.int32), sizes)


def part_random_balanced(n, K, rng):
    """Seeded permutation pi; part[pi[t]] = floor(t*K/n)."""
    pi = rng.permutation(n)
    part = np.empty(n, dtype=np.int32)
    t = np.arange(n, dtype=np.int64)
    part[pi] = (t * K // n).astype(np.int32)
    return part


def part_random_iid(n, K, rng):
    return rng.integers(0, K, size=n).astype(np.int32)


# --------------------------------------------------------------------------
# Matrix families
# --------------------------------------------------------------------------

def uniform_rows(n, per_row, rng):
    """Config 1: each row has `per_row` distinct uniform columns (diagonal not
    forced), values N(0,1) redrawn if exactly 0."""
    cols = np.empty((n, per_row), dtype=np.int64)
    chunk = max(1, (1 << 22) // max(n, 1))
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        keys = rng.random((r1 - r0, n))
        cols[r0:r1] = np.argpartition(keys, per_row - 1, axis=1)[:, :per_row]
    cols.sort(axis=1)
    vals = _nonzero_normal(rng, n * per_row).reshape(n, per_row)
    mask = np.ones((n, per_row), dtype=bool)
    return _rows_to_csr(n, cols, mask, vals)


def stencil2d(N, rng):
    """Config 2: 5-point stencil on an N x N grid, i = x*N + y, Dirichlet
    truncation; a_ii = 4 + U(0,1); off-diagonals -1 + U(-0.3, 0.3)."""
    n = N * N
    i = np.arange(n, dtype=np.int64)
    x, y = i // N, i % N
    diag = 4.0 + rng.uniform(0.0, 1.0, n)
    off = -1.0 + rng.uniform(-0.3, 0.3, (n, 4))
    # ascending column order: -N (x-1), -1 (y-1), 0, +1 (y+1), +N (x+1)
    cols = np.stack([i - N, i - 1, i, i + 1, i + N], axis=1)
    mask = np.stack([x > 0, y > 0, np.ones(n, bool), y < N - 1, x < N - 1], axis=1)
    vals = np.stack([off[:, 0], off[:, 1], diag, off[:, 2], off[:, 3]], axis=1)
    return _rows_to_csr(n, cols, mask, vals)


def stencil3d(N, rng):
    """Config 3: 7-point stencil on N^3, i = (x*N + y)*N + z, Dirichlet;
    off-diagonals -1, the +x neighbour -1 + u_i with u_i ~ U(0, 0.5);
    diagonal 6.0 (BASELINE leaves it unstated; SURVEY.md §8(d) D2 reading)."""
    n = N * N * N
    i = np.arange(n, dtype=np.int64)
    z = i % N
    y = (i // N) % N
    x = i // (N * N)
    u = rng.uniform(0.0, 0.5, n)
    NN = N * N
    cols = np.stack([i - NN, i - N, i - 1, i, i + 1, i + N, i + NN], axis=1)
    mask = np.stack([x > 0, y > 0, z > 0, np.ones(n, bool), z < N - 1, y < N - 1, x < N - 1], axis=1)
    m1 = np.full(n, -1.0)
    vals = np.stack([m1, m1, m1, np.full(n, 6.0), m1, m1, -1.0 + u], axis=1)
    del x, y, z
    return _rows_to_csr(n, cols, mask, vals)


def powerlaw(n, rng, alpha=2.1, kmax=5000, shift=0):
    """Config 4: row nnz k_i ~ Zipf(alpha) (+shift) clipped to [1, kmax]; row i
    = diagonal + (k_i - 1) distinct uniform off-diagonal columns; N(0,1)."""
    k = np.clip(rng.zipf(alpha, size=n) + shift, 1, min(kmax, n)).astype(np.int64)
    m = k - 1
    M = int(m.sum())
    rows = np.repeat(np.arange(n, dtype=np.int64), m)
    u = rng.integers(0, n - 1, size=M, dtype=np.int64)
    cols = u + (u >= rows)  # skip the diagonal
    while True:
        key = rows * n + cols
        order = np.argsort(key, kind="stable")
        ks = key[order]
        dup = np.zeros(M, dtype=bool)
        if M > 1:
            dup[order[1:][ks[1:] == ks[:-1]]] = True
        nd = int(dup.sum())
        if nd == 0:
            break
        u = rng.integers(0, n - 1, size=nd, dtype=np.int64)
        cols[dup] = u + (u >= rows[dup])
    rows = np.concatenate([rows, np.arange(n, dtype=np.int64)])
    cols = np.concatenate([cols, np.arange(n, dtype=np.int64)])
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    vals = _nonzero_normal(rng, rows.size)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return row_ptr, cols.astype(np.int32), vals


def banded(n, rng, bw=50, in_band=19, far=3, chunk=1 << 18):
    """Config 5: row i = diagonal + `in_band` distinct uniform columns with
    1 <= |i-j| <= bw + `far` distinct uniform columns with |i-j| > bw;
    off-diagonals U(-1,1); a_ii = 1 + sum_j |a_ij| (diagonally dominant)."""
    per = 1 + in_band + far
    offs = np.concatenate([np.arange(-bw, 0), np.arange(1, bw + 1)]).astype(np.int64)
    row_ptr = np.arange(n + 1, dtype=np.int64) * per
    col = np.empty(n * per, dtype=np.int32)
    val = np.empty(n * per, dtype=np.float64)
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        c = r1 - r0
        R = np.arange(r0, r1, dtype=np.int64)
        cand = R[:, None] + offs[None, :]
        valid = (cand >= 0) & (cand < n)
        keys = rng.random((c, offs.size))
        keys[~valid] = 2.0
        pick = np.argpartition(keys, in_band - 1, axis=1)[:, :in_band]
        band = np.take_along_axis(cand, pick, axis=1)
        lo = np.maximum(R - bw, 0)
        hi = np.minimum(R + bw, n - 1)
        allowed = n - (hi - lo + 1)
        fars = np.empty((c, far), dtype=np.int64)
        for t in range(far):
            fars[:, t] = rng.integers(0, allowed)
        while True:
            dup = np.zeros((c, far), dtype=bool)
            for a in range(far):
                for b in range(a):
                    dup[:, a] |= fars[:, a] == fars[:, b]
            nd = int(dup.sum())
            if nd == 0:
                break
            rr = np.nonzero(dup)[0]
            fars[dup] = rng.integers(0, allowed[rr])
        fars = np.where(fars < lo[:, None], fars, fars + (hi - lo + 1)[:, None])
        offv = _nonzero_uniform(rng, -1.0, 1.0, c * (in_band + far)).reshape(c, in_band + far)
        diag = 1.0 + np.abs(offv).sum(axis=1)
        cols = np.concatenate([R[:, None], band, fars], axis=1)
        vals = np.concatenate([diag[:, None], offv], axis=1)
        order = np.argsort(cols, axis=1)
        cols = np.take_along_axis(cols, order, axis=1)
        vals = np.take_along_axis(vals, order, axis=1)
        col[r0 * per:r1 * per] = cols.reshape(-1)
        val[r0 * per:r1 * per] = vals.reshape(-1)
    return row_ptr, col, val


def dense_rows(n, rng, per_row=64, bw=1000):
    """Config 7: row i = diagonal + (per_row - 1) distinct
    uniform columns with 1 <= |i-j| <= bw (clipped to the matrix); U(-1,1)
    off-diagonals, diagonal 1 + sum |off| -- FEM-like rows of nnz/n ~ 64, the
    regime of the paper's largest-nnz matrices."""
    offs = np.concatenate([np.arange(-bw, 0), np.arange(1, bw + 1)]).astype(np.int64)
    m = per_row - 1
    R = np.arange(n, dtype=np.int64)
    cand = R[:, None] + offs[None, :]
    valid = (cand >= 0) & (cand < n)
    keys = rng.random((n, offs.size))
    keys[~valid] = 2.0
    pick = np.argpartition(keys, m - 1, axis=1)[:, :m]
    cols = np.take_along_axis(cand, pick, axis=1)
    ok = np.take_along_axis(valid, pick, axis=1)
    offv = _nonzero_uniform(rng, -1.0, 1.0, n * m).reshape(n, m)
    offv[~ok] = 0.0
    cols[~ok] = -1
    diag = 1.0 + np.abs(offv).sum(axis=1)
    cols = np.concatenate([R[:, None], cols], axis=1)
    vals = np.concatenate([diag[:, None], offv], axis=1)
    mask = cols >= 0
    order = np.argsort(np.where(mask, cols, np.iinfo(np.int64).max), axis=1)
    cols = np.take_along_axis(cols, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    mask = np.take_along_axis(mask, order, axis=1)
    return _rows_to_csr(n, cols, mask, vals)


def dense_columns(n, rng, per_row=5, n_dense=4, dense_nnz=None, ncols=None, levels=0):
    """Sparse rows plus planted dense columns (the LP-matrix shape that
    motivates the sparsification of PAPER.md:565-576): every row has
    `per_row` distinct uniform columns, and `n_dense` evenly spaced columns
    hold `dense_nnz` (default n // 4) uniformly chosen rows each.  Values
    N(0,1), or with `levels` > 0 drawn from {+-1, ..., +-levels} so that
    |value| ties are common (the tie rule of SPEC.md:229)."""
    m = n if ncols is None else int(ncols)
    dense_nnz = n // 4 if dense_nnz is None else int(dense_nnz)
    dcols = (np.arange(n_dense, dtype=np.int64) * m) // max(n_dense, 1) + m // (2 * max(n_dense, 1))
    rows = [np.repeat(np.arange(n, dtype=np.int64), per_row)]
    keys = rng.random((n, m)) if n * m <= (1 << 24) else None
    if keys is not None:
        keys[:, dcols] = 2.0  # the dense columns come from their own draw
        cols = [np.sort(np.argpartition(keys, per_row - 1, axis=1)[:, :per_row], axis=1).reshape(-1)]
    else:
        free = np.delete(np.arange(m, dtype=np.int64), dcols)  # the non-dense columns
        t = np.sort(rng.integers(0, free.size, size=(n, per_row)), axis=1)
        while True:
            dup = np.zeros_like(t, dtype=bool)
            dup[:, 1:] = t[:, 1:] == t[:, :-1]
            if not dup.any():
                break
            t[dup] = rng.integers(0, free.size, size=int(dup.sum()))
            t.sort(axis=1)
        cols = [free[t].reshape(-1)]
    for k in dcols:
        r = np.sort(rng.choice(n, size=dense_nnz, replace=False))
        rows.append(r)
        cols.append(np.full(r.size, k, dtype=np.int64))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    if levels > 0:
        vals = rng.integers(1, levels + 1, size=rows.size) * rng.choice([-1.0, 1.0], size=rows.size)
    else:
        vals = _nonzero_normal(rng, rows.size)
    return from_triplets(n, m, rows, cols, vals)


# --------------------------------------------------------------------------
# BASELINE.json configs
# --------------------------------------------------------------------------

FULL = {1: 2000, 2: 1000, 3: 200, 4: 2_000_000, 5: 4_000_000, 6: 2_000_000, 7: 100_000}
# reduced twins: same recipe, sizes the oracle finishes in seconds while still
# spanning many tiles/CTAs and a ragged tail
SMALL = {1: 2000, 2: 151, 3: 23, 4: 40_001, 5: 30_011, 6: 20_011, 7: 3_001}


def make(cfg_id: int, size=None) -> Workload:
    """Build BASELINE.json config `cfg_id` (1-based).  `size` overrides the
    grid side (cfgs 2, 3) or n (cfgs 1, 4, 5)."""
    cfg_id = int(cfg_id)
    size = FULL[cfg_id] if size is None else int(size)
    rng = np.random.default_rng(SEED_BASE + cfg_id)
    prng = np.random.default_rng(SEED_BASE + 1000 + cfg_id)
    if cfg_id == 1:
        n = size
        rp, ci, v = uniform_rows(n, 5, rng)
        scale, tol, K = 1, 0.0, 4
        part = part_contiguous(n, K)
        recipe = f"n={n}, 5 distinct uniform cols/row, N(0,1), scaled, drop_tol=0, K=4 contiguous"
    elif cfg_id == 2:
        n = size * size
        rp, ci, v = stencil2d(size, rng)
        scale, tol, K = 1, 0.0, 8
        part = part_contiguous(n, K)
        recipe = f"{size}x{size} 5-point stencil, diag 4+U(0,1), off -1+U(-.3,.3), scaled, drop_tol=0, K=8 contiguous"
    elif cfg_id == 3:
        n = size ** 3
        rp, ci, v = stencil3d(size, rng)
        scale, tol, K = 1, 1e-8, 64
        part = part_random_balanced(n, K, prng)
        recipe = f"{size}^3 7-point stencil, off -1, +x -1+U(0,.5), diag 6, scaled, drop_tol=1e-8, K=64 random-balanced"
    elif cfg_id == 4:
        n = size
        rp, ci, v = powerlaw(n, rng)
        scale, tol, K = 1, 0.0, 128
        part = part_random_iid(n, K, prng)
        recipe = f"n={n}, row nnz ~ Zipf(2.1) clipped [1,5000], diag forced, N(0,1), scaled, drop_tol=0, K=128 iid"
    elif cfg_id == 5:
        n = size
        rp, ci, v = banded(n, rng)
        scale, tol, K = 0, 1e-6, 256
        part = part_contiguous(n, K)
        recipe = f"n={n}, bw 50: 19 in-band + 3 far cols/row, U(-1,1), diag 1+sum|off|, unscaled, drop_tol=1e-6, K=256 contiguous"
    elif cfg_id == 6:  # SURVEY §8(f) f3 / §8(d) D2 "4-alt": BASELINE's "mean ~12"
        n = size
        rp, ci, v = powerlaw(n, rng, shift=8)
        scale, tol, K = 1, 0.0, 128
        part = part_random_iid(n, K, prng)
        recipe = f"n={n}, row nnz ~ Zipf(2.1)+8 clipped [1,5000] (mean ~12.3), diag forced, N(0,1), scaled, drop_tol=0, K=128 iid"
    elif cfg_id == 7:  # dense rows
        n = size
        rp, ci, v = dense_rows(n, rng)
        scale, tol, K = 1, 0.0, 32
        part = part_contiguous(n, K)
        recipe = f"n={n}, 64 entries/row: diag + 63 uniform cols with |i-j|<=1000, U(-1,1), diag 1+sum|off|, scaled, drop_tol=0, K=32 contiguous"
    else:
        raise ValueError(f"unknown config {cfg_id}")
    return Workload(CONFIG_NAMES[cfg_id], cfg_id, n, n, rp, ci, v, scale, tol, part, K, recipe)


def make_small(cfg_id: int) -> Workload:
    return make(cfg_id, SMALL[int(cfg_id)])
