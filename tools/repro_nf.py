"""Small edge-case builds in a fresh process each (debugging aid): python tools/repro_nf.py CASE"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1710_07769_b200 import rig  # noqa: E402

case = sys.argv[1]
if case == "nonsq_inf":
    A = rig.CSR(np.array([0, 2, 3]), np.array([0, 1, 2], np.int32), np.array([1.0, np.inf, 3.0]), ncols=3)
elif case == "nonsq":
    A = rig.CSR(np.array([0, 2, 3]), np.array([0, 1, 2], np.int32), np.array([1.0, 2.0, 3.0]), ncols=3)
elif case == "sq_inf":
    A = rig.CSR(np.array([0, 2, 3]), np.array([0, 1, 1], np.int32), np.array([1.0, np.inf, 3.0]))
elif case == "sq":
    A = rig.CSR(np.array([0, 2, 3]), np.array([0, 1, 1], np.int32), np.array([1.0, 2.0, 3.0]))
for sc in (1, 0):
    try:
        g = rig.rig_build(A, sc, 0.0)
        print(case, sc, "ok", g.n, g.nnz)
    except rig.RigError as e:
        print(case, sc, "err", e.code, e)
