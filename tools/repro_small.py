"""Build one small config through the C ABI (debugging aid)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1710_07769_b200 import rig  # noqa: E402
from rig_inputs import make_small  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = make_small(cfg)
A = rig.CSR(w.row_ptr, w.col_idx, w.val)
g = rig.rig_build(A, w.scale_rows, w.drop_tol, rig.RIG_FLAG_DIAG)
torch.cuda.synchronize()
print("ok", g.n, g.nnz)
