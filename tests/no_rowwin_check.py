"""Run by test_gpu_parity.test_without_row_window in a fresh process with
RIG_ROWWIN=0: the path a matrix takes when the row-window kernel cannot
(n >= 2^25 rows, or CSC offsets beyond int32) -- mid rows through the older
passes (window + far list of 256 / 768 items, wide window, global far lists)
and the CTA accumulator kernel.  Every graph, diagonal and cut must equal the
oracle (graph bit for bit, cut within 1e-12)."""
import numpy as np
import torch

import oracle
from paper_1710_07769_b200 import rig
from rig_inputs import from_triplets, make_small


def check(rp, ci, v, scale, tol, part, K):
    orc = oracle.build(rp, ci, v, scale_rows=scale, drop_tol=tol)
    A = rig.CSR(rp, ci, v)
    g = rig.rig_build(A, scale, tol, rig.RIG_FLAG_DIAG)
    torch.cuda.synchronize()
    assert rig.last_path() != "rowwin", rig.last_path()
    assert np.array_equal(g.row_ptr.cpu().numpy(), orc.row_ptr)
    assert np.array_equal(g.col_idx.cpu().numpy(), orc.col)
    assert g.w.cpu().numpy().tobytes() == orc.w.tobytes()
    assert g.diag.cpu().numpy().tobytes() == orc.diag.tobytes()
    ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, part, K)[0]
    n = len(rp) - 1
    _, cut = rig.rig_build_cut(A, torch.as_tensor(part, device="cuda"), K, 0, n, scale, tol)
    assert abs(cut.item() - ocut) <= 1e-12 * max(ocut, 1e-300)
    return rig.last_path()


def main():
    paths = set()
    for cfg in (4, 5, 6, 7):  # mixed skew, banded, power law, dense rows
        w = make_small(cfg)
        paths.add(check(w.row_ptr, w.col_idx, w.val, w.scale_rows, w.drop_tol, w.part, w.K))
    rng = np.random.default_rng(11)
    n = 4000
    lens = np.clip(rng.zipf(1.6, n), 1, 1500)  # a few very long rows: far lists beyond 768 items
    rows = np.repeat(np.arange(n), lens)
    cols = rng.integers(0, n, rows.size)
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    vals[rng.random(rows.size) < 0.3] = 1.0
    rp, ci, v = from_triplets(n, n, rows, cols, vals)
    part = rng.integers(0, 9, n).astype(np.int32)
    for scale, tol in ((1, 0.0), (0, 0.5)):
        paths.add(check(rp, ci, v, scale, tol, part, 9))
    print("no-rowwin paths ok", sorted(paths))


if __name__ == "__main__":
    main()
