"""Long rows of scattered columns on the mixed path: the CTA kernel's key-range
launch (k_row_cta<RANGE>: rows beyond its shared arrays in ranges of
consecutive key buckets, warp per range; crowded buckets split by the next
key bits) and what falls past it (a key with more products than a warp range
holds: the global-far-list and CTA-accumulator kernels, with their scratch
allocated on demand).  Every graph must equal the oracle bit for bit.

Run in-process by test_gpu_parity.test_long_rows_key_ranges, and in fresh
processes with RIG_LONG_SCRATCH_MB overrides (slices too small for the
longest rows: a mixture; no range launch at all)."""
import numpy as np
import torch

import oracle
from paper_1710_07769_b200 import rig
from rig_inputs import from_triplets


def long_rows_matrix(seed):
    """n = 40000: rows of 1..5 random columns; every 997th row 300..1500
    columns (f_i ~ 1.5k..9k: one to several key ranges); rows 0..255 (the
    first key bucket) all hold the 20 columns 1000..1019, so each of them has
    >= 5100 products in one bucket (a crowded bucket: split by the next key
    bits); rows 300 and 301 share 900 columns (900 products of one key: the
    fallback chain).  Values with exact ties (+-1) force cancellations and
    equal-key groups."""
    rng = np.random.default_rng(seed)
    n = 40000
    rows, cols = [], []
    for r in range(n):
        k = int(rng.integers(300, 1500)) if r % 997 == 3 else int(rng.integers(1, 6))
        cc = rng.choice(n, k, replace=False)
        rows.append(np.full(k, r)); cols.append(cc)
    blk = np.arange(256)
    dense = np.arange(1000, 1020)
    rows.append(np.repeat(blk, dense.size)); cols.append(np.tile(dense, blk.size))
    shared = rng.choice(n, 900, replace=False)
    rows += [np.full(900, 300), np.full(900, 301)]; cols += [shared, shared]
    rows.append(np.arange(n)); cols.append(np.arange(n))
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    vals[rng.random(rows.size) < 0.2] = 1.0
    vals[rng.random(rows.size) < 0.2] = -1.0
    return n, from_triplets(n, n, rows, cols, vals)


def run(seed=0):
    n, (rp, ci, v) = long_rows_matrix(seed)
    A = rig.CSR(rp, ci, v)
    K = 32
    part = np.random.default_rng(seed + 1).integers(0, K, n).astype(np.int32)
    tpart = torch.as_tensor(part, device="cuda")
    for scale, tol in ((1, 0.0), (0, 0.7)):
        orc = oracle.build(rp, ci, v, scale_rows=scale, drop_tol=tol)
        g, cut = rig.rig_build_cut(A, tpart, K, 0, n, scale, tol, flags=rig.RIG_FLAG_DIAG)
        torch.cuda.synchronize()
        assert rig.last_path() == "mixed", rig.last_path()
        assert np.array_equal(g.row_ptr.cpu().numpy(), orc.row_ptr)
        assert np.array_equal(g.col_idx.cpu().numpy(), orc.col)
        assert g.w.cpu().numpy().tobytes() == orc.w.tobytes()
        assert g.diag.cpu().numpy().tobytes() == orc.diag.tobytes()
        ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, part, K)[0]
        assert abs(cut.item() - ocut) <= 1e-12 * abs(ocut), (cut.item(), ocut)
    # a shard that starts inside the dense block and ends past a long row
    a, b = 100, 30000
    o3 = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0, row_begin=a, row_end=b)
    g3 = rig.rig_build_rows(A, a, b, 1, 0.0)
    assert np.array_equal(g3.row_ptr.cpu().numpy(), o3.row_ptr)
    assert np.array_equal(g3.col_idx.cpu().numpy(), o3.col)
    assert g3.w.cpu().numpy().tobytes() == o3.w.tobytes()


if __name__ == "__main__":
    run(0)
    print("long rows ok")
