"""Whole-graph parity at BASELINE.json's full sizes (configs 1-5), in the
launch configuration bench.py times (rig_build_cut over all rows), against
the oracle's graph recorded as sha256 digests of fixed row blocks in
tests/golden/full_size_digests.json (written by tools/make_full_golden.py,
which calls only oracle/).  Bar (BASELINE.json north_star): row_ptr and
col_idx bit-exact, weights within 1e-12 relative -- a digest match is bit
equality of row_ptr, col, w and diag together; cutsize within 1e-12 relative.

On a digest mismatch the oracle recomputes that block and the test reports
the first differing element.
"""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import oracle  # noqa: E402
from rig_inputs import make  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "full_size_digests.json")
REL = 1e-12


@pytest.fixture(scope="module")
def rig():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1710_07769_b200 import rig as r

    return r


def _input_digest(w):
    h = hashlib.sha256()
    for a in (w.row_ptr, w.col_idx, w.val, w.part):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _digest(rp_local, col, wv, diag):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rp_local, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(col, dtype="<i4").tobytes())
    h.update(np.ascontiguousarray(wv, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(diag, dtype="<f8").tobytes())
    return h.hexdigest()


def _explain(w, a, b, rp, col, wv, diag):
    a_hat = oracle.scale(w.row_ptr, w.val)[0] if w.scale_rows else w.val
    csc = oracle.transpose(w.n, w.ncols, w.row_ptr, w.col_idx, a_hat)
    o_rp, o_col, o_w, o_diag, _ = oracle.build_from_scaled(w.n, w.ncols, w.row_ptr, w.col_idx, a_hat, csc,
                                                           w.drop_tol, a, b, threads=oracle.default_threads())
    for name, x, y in (("row_ptr", rp, o_rp), ("col", col, o_col), ("w", wv, o_w), ("diag", diag, o_diag)):
        if x.shape != y.shape:
            return f"{name}: shape {x.shape} vs oracle {y.shape}"
        xi = x.view(np.int64) if x.dtype == np.float64 else x  # bitwise for weights
        yi = y.view(np.int64) if y.dtype == np.float64 else y
        bad = np.nonzero(xi != yi)[0]
        if bad.size:
            k = int(bad[0])
            return f"{name}[{k}] = {x[k]!r}, oracle {y[k]!r} ({bad.size} differ)"
    return "digests differ but no element does (hash input mismatch)"


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_full_size_whole_graph(rig, cfg):
    with open(GOLD) as fh:
        gold = json.load(fh).get(str(cfg))
    if gold is None:
        pytest.fail(f"no golden digests for config {cfg}: run tools/make_full_golden.py")
    w = make(cfg)
    assert _input_digest(w) == gold["input_sha256"], "input generator drifted from the golden record"
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    part = torch.as_tensor(w.part, device="cuda")
    g, cut = rig.rig_build_cut(A, part, w.K, 0, w.n, w.scale_rows, w.drop_tol, flags=rig.RIG_FLAG_DIAG)
    torch.cuda.synchronize()
    assert g.nnz == gold["graph_nnz"]
    rp_all = g.row_ptr.cpu().numpy()
    diag_all = g.diag.cpu().numpy()
    for blk in gold["blocks"]:
        a, b = blk["rows"]
        s, e = int(rp_all[a]), int(rp_all[b])
        assert e - s == blk["nnz"], f"rows [{a},{b}): {e - s} edges, oracle {blk['nnz']}"
        rp = rp_all[a:b + 1] - s
        col = g.col_idx[s:e].cpu().numpy()
        wv = g.w[s:e].cpu().numpy()
        diag = diag_all[a:b]
        if _digest(rp, col, wv, diag) != blk["sha256"]:
            pytest.fail(f"config {cfg} rows [{a},{b}): {_explain(w, a, b, rp, col, wv, diag)}")
    c = cut.item()
    assert abs(c - gold["cut"]) <= REL * abs(gold["cut"]), (c, gold["cut"])
    del g
    torch.cuda.empty_cache()
