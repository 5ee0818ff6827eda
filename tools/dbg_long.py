"""Debug: rows of make_small(4) (or the long-rows matrix) whose graph row differs from the oracle."""
import sys
import numpy as np
import torch
import oracle
from paper_1710_07769_b200 import rig
from rig_inputs import make_small
sys.path.insert(0, "tests")

if sys.argv[1] == "long":
    import long_rows_check
    n, (rp, ci, v) = long_rows_check.long_rows_matrix(0)
    scale, tol = 1, 0.0
else:
    w = make_small(int(sys.argv[1]))
    n, rp, ci, v, scale, tol = w.n, w.row_ptr, w.col_idx, w.val, w.scale_rows, w.drop_tol
cl = np.bincount(ci, minlength=n).astype(np.int64)
ln = np.diff(rp)
f = np.add.reduceat(cl[ci], rp[:-1]) * (ln > 0)
orc = oracle.build(rp, ci, v, scale_rows=scale, drop_tol=tol)
for a, b in ((0, n), (0, n // 2), (n // 2, n)):
    g = rig.rig_build_rows(rig.CSR(rp, ci, v), a, b, scale, tol)
    torch.cuda.synchronize()
    print("rows", a, b, "path", rig.last_path())
    o = oracle.build(rp, ci, v, scale_rows=scale, drop_tol=tol, row_begin=a, row_end=b)
    grp, gc, gw = g.row_ptr.cpu().numpy(), g.col_idx.cpu().numpy(), g.w.cpu().numpy()
    if not np.array_equal(grp, o.row_ptr):
        bad = np.flatnonzero(np.diff(grp) != np.diff(o.row_ptr))
        print(" row_ptr differs in", bad.size, "rows; first", bad[:10] + a, "f", f[bad[:10] + a])
        continue
    badr = []
    for r in range(b - a):
        s, e = grp[r], grp[r + 1]
        if not (np.array_equal(gc[s:e], o.col[s:e]) and gw[s:e].tobytes() == o.w[s:e].tobytes()):
            badr.append(r)
    print(" rows differing:", len(badr), "f:", [int(f[r + a]) for r in badr[:20]], "len:", [int(ln[r + a]) for r in badr[:20]])
    for r in badr[:2]:
        s, e = grp[r], grp[r + 1]
        print("  row", r + a, "gpu", gc[s:s + 12], "orc", o.col[s:s + 12])
        d = np.flatnonzero(gc[s:e] != o.col[s:e])
        print("  first diff at", d[:5], "of", e - s)
