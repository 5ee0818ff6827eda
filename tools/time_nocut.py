"""Numeric-kernel time of config C with and without the fused cut (profiling aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1710_07769_b200 import rig  # noqa: E402
from rig_inputs import make  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = make(c)
A = rig.CSR(w.row_ptr, w.col_idx, w.val)
part = torch.as_tensor(w.part, device="cuda")
import ctypes  # noqa: E402
ms = (ctypes.c_double * 16)()
cnt = (ctypes.c_int64 * 16)()
for mode in ("cut", "nocut", "cut", "nocut"):
    rig.lib.rig_profile_enable(1)
    rig.lib.rig_profile_read(None, None)
    for _ in range(10):
        if mode == "cut":
            g, cut = rig.rig_build_cut(A, part, w.K, 0, w.n, w.scale_rows, w.drop_tol)
        else:
            g = rig.rig_build(A, w.scale_rows, w.drop_tol, 0)
        del g
    torch.cuda.synchronize()
    rig.lib.rig_profile_read(ms, cnt)
    print(mode, {rig.lib.rig_pass_name(i).decode(): round(ms[i] / 10, 4) for i in range(13) if cnt[i]})
