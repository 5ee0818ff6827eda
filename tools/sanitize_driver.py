"""Exercise every librig kernel path on small inputs (for compute-sanitizer).

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_07769_b200 import rig  # noqa: E402
from rig_inputs import from_triplets, make_small  # noqa: E402


def mixed(n, seed):
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    c0 = rng.choice(n, min(3000, n // 2), replace=False)
    rows += [0] * c0.size
    cols += list(c0)
    for r in range(1, 60):
        k = int(rng.integers(9, 400))
        cc = rng.choice(n, k, replace=False)
        rows += [r] * k
        cols += list(cc)
    rows += list(range(n))
    cols += list(rng.integers(0, n, n))
    r7 = rng.choice(np.arange(60, n), min(600, n - 60), replace=False)
    rows += list(r7)
    cols += [7] * r7.size
    key = np.unique(np.array(rows, np.int64) * n + np.array(cols, np.int64))
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    return from_triplets(n, n, rows, cols, vals)


def main():
    torch.cuda.set_device(0)
    for cfg in (1, 2, 3, 4, 5):
        w = make_small(cfg)
        A = rig.CSR(w.row_ptr, w.col_idx, w.val)
        part = torch.as_tensor(w.part, device="cuda")
        g, cut = rig.rig_build_cut(A, part, w.K, 0, w.n, w.scale_rows, w.drop_tol, rig.RIG_FLAG_DIAG)
        rig.rig_cutsize(g, part, w.K)
        p = rig.Plan(A, w.scale_rows, w.drop_tol, rig.RIG_FLAG_DIAG)
        p.execute()
        p.destroy()
        sp = rig.rig_row_split(A, 3)
        rig.rig_build_rows(A, sp[1], sp[2], w.scale_rows, w.drop_tol)
        # holes path
        rig.rig_build_cut(A, part, w.K, 0, w.n, w.scale_rows, 0.3 if w.scale_rows else 2.0)
        torch.cuda.synchronize()
        print("cfg", cfg, "ok", g.nnz, float(cut.item()))
    rp, ci, v = mixed(5000, 1)
    A = rig.CSR(rp, ci, v)
    part = torch.zeros(5000, dtype=torch.int32, device="cuda")
    g, cut = rig.rig_build_cut(A, part, 1, 0, 5000, 1, 0.0, rig.RIG_FLAG_DIAG)
    g2 = rig.rig_build(A, 1, 0.05, rig.RIG_FLAG_VALIDATE)
    torch.cuda.synchronize()
    print("mixed ok", g.nnz, g2.nnz)
    # row-window path: every row off the merge path; random rows take the
    # global far list (and the capacity retry), banded rows the window
    rng = np.random.default_rng(3)
    n = 3000
    rows, cols = [], []
    for r in range(n):
        if r < n // 2:
            cc = rng.choice(n, int(rng.integers(9, 31)), replace=False)
        else:
            cc = np.unique(np.concatenate([[r], np.clip(r + rng.integers(-60, 61, 20), 0, n - 1),
                                           rng.integers(0, n, 2)]))
        rows += [r] * cc.size
        cols += list(cc)
    key = np.unique(np.array(rows, np.int64) * n + np.array(cols, np.int64))
    rows, cols = key // n, key % n
    rp, ci, v = from_triplets(n, n, rows, cols, rng.standard_normal(rows.size))
    A = rig.CSR(rp, ci, v)
    part = torch.as_tensor(rng.integers(0, 8, n).astype(np.int32), device="cuda")
    g, cut = rig.rig_build_cut(A, part, 8, 0, n, 1, 0.0, rig.RIG_FLAG_DIAG)
    torch.cuda.synchronize()
    print("rowwin ok", g.nnz, rig.last_path(), float(cut.item()))


if __name__ == "__main__":
    main()
