import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle
from rig_inputs import from_triplets
from paper_1710_07769_b200 import rig
seed=int(sys.argv[1]) if len(sys.argv)>1 else 0
rng = np.random.default_rng(900 + seed)
n = 5000
rows, cols = [], []
for r in range(n):
    if r < n // 2:
        cc = rng.choice(n, int(rng.integers(9, 31)), replace=False)
    else:
        cc = np.unique(np.concatenate([[r], np.clip(r + rng.integers(-60, 61, 20), 0, n - 1), rng.integers(0, n, 2)]))
    rows += [r] * cc.size; cols += list(cc)
rows, cols = np.array(rows), np.array(cols)
key = np.unique(rows.astype(np.int64) * n + cols)
rows, cols = key // n, key % n
vals = rng.standard_normal(rows.size)
vals[rng.random(rows.size) < 0.2] = 1.0
vals[rng.random(rows.size) < 0.2] = -1.0
rp, ci, v = from_triplets(n, n, rows, cols, vals)
A = rig.CSR(rp, ci, v)
orc = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0)
g = rig.rig_build(A, 1, 0.0, rig.RIG_FLAG_DIAG)
grp = g.row_ptr.cpu().numpy(); gcol = g.col_idx.cpu().numpy(); gw = g.w.cpu().numpy()
cnt_g = np.diff(grp); cnt_o = np.diff(orc.row_ptr)
bad = np.nonzero(cnt_g != cnt_o)[0]
print("rows with wrong count:", bad.size, bad[:10])
cl = np.bincount(ci, minlength=n)
for r in bad[:5]:
    ks = ci[rp[r]:rp[r+1]]
    U = int(((cl[ks] + 31)//32).sum())
    print("row", r, "len", ks.size, "U", U, "gpu", cnt_g[r], "orc", cnt_o[r])
    a = set(gcol[grp[r]:grp[r+1]].tolist()); b = set(orc.col[orc.row_ptr[r]:orc.row_ptr[r+1]].tolist())
    print("  missing", sorted(b-a)[:10], "extra", sorted(a-b)[:10])
# per-row values for matching count rows
ok = np.nonzero(cnt_g == cnt_o)[0]
