"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by
element on the same seeded inputs.

Bar (BASELINE.json north_star): graph row_ptr / col_idx bit-exact; weights
and cutsize within 1e-12 relative.  Under the ordering contract (DESIGN.md §3
R4) the weights are expected bit-identical, so that is asserted too.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from rig_inputs import from_dense, from_triplets, make, make_small  # noqa: E402

REL = 1e-12


@pytest.fixture(scope="module")
def rig():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1710_07769_b200 import rig as r

    return r


def to_np(t):
    return t.detach().cpu().numpy()


def assert_graph_equal(g_rp, g_col, g_w, orc, g_diag=None, bitwise=True):
    np.testing.assert_array_equal(g_rp, orc.row_ptr)
    np.testing.assert_array_equal(g_col, orc.col)
    if orc.w.size:
        rel = np.abs(g_w - orc.w) / np.abs(orc.w)
        assert rel.max() <= REL, f"max rel err {rel.max()}"
    if bitwise:
        assert g_w.tobytes() == orc.w.tobytes(), f"{int((g_w != orc.w).sum())} weights differ in bits"
    if g_diag is not None:
        assert g_diag.tobytes() == orc.diag.tobytes()


def gpu_build(rig, w, flags=None, **kw):
    A = rig.CSR(w.row_ptr, w.col_idx, w.val, ncols=w.ncols)
    g = rig.rig_build(A, w.scale_rows, w.drop_tol, rig.RIG_FLAG_DIAG if flags is None else flags, **kw)
    return A, g


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6, 7])
def test_small_configs_bitexact(rig, cfg):
    w = make_small(cfg)
    orc = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol)
    A, g = gpu_build(rig, w)
    assert g.n == w.n and g.nnz == orc.nnz
    assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc, to_np(g.diag))
    part = torch.as_tensor(w.part, device="cuda")
    cut = rig.rig_cutsize(g, part, w.K).item()
    ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, w.part, w.K)[0]
    assert abs(cut - ocut) <= REL * abs(ocut)
    # staged API gives the same graph
    plan = rig.Plan(A, w.scale_rows, w.drop_tol, rig.RIG_FLAG_DIAG)
    assert plan.products == orc.products
    tg = plan.execute()
    assert_graph_equal(to_np(tg.row_ptr), to_np(tg.col_idx), to_np(tg.w), orc, to_np(tg.diag))
    plan.destroy()


@pytest.mark.parametrize("cfg", [1, 3, 5])
def test_build_cut_fused(rig, cfg):
    """rig_build_cut (cutsize enqueued on the upper-bound layout) == oracle."""
    w = make_small(cfg)
    orc = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol)
    ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, w.part, w.K)[0]
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    part = torch.as_tensor(w.part, device="cuda")
    g, cut = rig.rig_build_cut(A, part, w.K, 0, w.n, w.scale_rows, w.drop_tol)
    assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc)
    assert abs(cut.item() - ocut) <= REL * ocut
    # holes (dropped entries) before the compaction: the cut must skip them
    tol = float(np.quantile(orc.w, 0.3))
    orc2 = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=tol)
    ocut2 = oracle.cutsize(orc2.row_ptr, orc2.col, orc2.w, w.part, w.K)[0]
    g2, cut2 = rig.rig_build_cut(A, part, w.K, 0, w.n, w.scale_rows, tol)
    assert_graph_equal(to_np(g2.row_ptr), to_np(g2.col_idx), to_np(g2.w), orc2)
    assert abs(cut2.item() - ocut2) <= REL * ocut2
    # a shard
    a, b = w.n // 3, 2 * w.n // 3
    o3 = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol, row_begin=a,
                      row_end=b)
    oc3 = oracle.cutsize(o3.row_ptr, o3.col, o3.w, w.part, w.K, row_begin=a)[0]
    g3, cut3 = rig.rig_build_cut(A, part, w.K, a, b, w.scale_rows, w.drop_tol)
    assert_graph_equal(to_np(g3.row_ptr), to_np(g3.col_idx), to_np(g3.w), o3)
    assert abs(cut3.item() - oc3) <= REL * oc3


def test_shards_concatenate_bitwise(rig):
    w = make_small(5)
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    full = rig.rig_build(A, w.scale_rows, w.drop_tol)
    split = rig.rig_row_split(A, 3)
    assert split[0] == 0 and split[-1] == w.n and all(a <= b for a, b in zip(split, split[1:]))
    f, P = oracle.row_products(w.row_ptr, w.col_idx, oracle.transpose(w.n, w.n, w.row_ptr, w.col_idx, w.val)[0])
    pre = np.concatenate([[0], np.cumsum(f)])
    for gi in range(4):  # split[g] = first r with prefix[r] >= ceil(g P / 3)
        if gi < 3:
            tgt = -(-gi * P // 3)
            assert split[gi] == int(np.searchsorted(pre, tgt, side="left"))
    cols, ws, cuts = [], [], []
    part = torch.as_tensor(w.part, device="cuda")
    for a, b in zip(split[:-1], split[1:]):
        s = rig.rig_build_rows(A, a, b, w.scale_rows, w.drop_tol)
        cols.append(to_np(s.col_idx)); ws.append(to_np(s.w))
        cuts.append(rig.rig_cutsize(s, part, w.K).item())
    np.testing.assert_array_equal(np.concatenate(cols), to_np(full.col_idx))
    assert np.concatenate(ws).tobytes() == to_np(full.w).tobytes()
    c_full = rig.rig_cutsize(full, part, w.K).item()
    assert abs(sum(cuts) - c_full) <= REL * c_full


def _dense_case(rig, D, scale, tol=0.0):
    rp, ci, v = from_dense(D)
    orc = oracle.build(rp, ci, v, ncols=D.shape[1], scale_rows=scale, drop_tol=tol)
    A = rig.CSR(rp, ci, v, ncols=D.shape[1])
    g = rig.rig_build(A, scale, tol, rig.RIG_FLAG_DIAG)
    assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc, to_np(g.diag) if g.n else None)
    return g, orc


def test_edge_cases(rig):
    # paper worked example c_24 = 216, unscaled
    D = np.zeros((8, 8)); D[1, 2] = 9; D[1, 6] = 6; D[3, 2] = 12; D[3, 6] = 18; D[0, 0] = 5; D[2, 1] = 4
    g, _ = _dense_case(rig, D, 0)
    G = np.zeros((8, 8))
    rp, c, wv = to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w)
    for r in range(8):
        G[r, c[rp[r]:rp[r + 1]]] = wv[rp[r]:rp[r + 1]]
    assert G[1, 3] == 216.0 and G[3, 1] == 216.0
    # exact cancellation -> no edge; drop rule strict
    D = np.array([[1.0, 1.0, 0], [1.0, -1.0, 0], [0, 0, 2.0]])
    g, orc = _dense_case(rig, D, 0)
    assert g.nnz == 0
    D = np.array([[1.0, 0.0], [0.5, 1.0]])
    assert _dense_case(rig, D, 0, 0.5)[0].nnz == 0
    assert _dense_case(rig, D, 0, np.nextafter(0.5, 0))[0].nnz == 2
    # duplicate rows, one-row, empty rows (unscaled), rectangular
    _dense_case(rig, np.array([[1.0, 2.0, 0.0], [1.0, 2.0, 0.0], [0.0, 0.0, 3.0]]), 1)
    _dense_case(rig, np.array([[3.0, 4.0]]), 1)
    _dense_case(rig, np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 2.0], [0.0, 0.0, 0.0]]), 0)
    rng = np.random.default_rng(5)
    D = (rng.random((50, 80)) < 0.1) * rng.standard_normal((50, 80))
    D[np.arange(50), rng.integers(0, 80, 50)] = 1.5
    _dense_case(rig, D, 1)
    # paper's dense-column example: nnz(AA^T) = 531
    D = np.eye(25)
    for r in range(25):
        if r not in (2, 19):
            D[r, 11] = 1.0 + r / 7.0
    g, orc = _dense_case(rig, D, 1)
    assert g.nnz == 506


def test_empty_and_errors(rig):
    A = rig.CSR(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    g = rig.rig_build(A, 0, 0.0)
    assert g.n == 0 and g.nnz == 0
    A = rig.CSR(np.array([0, 2, 2, 3]), np.array([0, 1, 2], np.int32), np.array([1.0, 2.0, 3.0]))
    with pytest.raises(rig.RigError) as e:
        rig.rig_build(A, 1, 0.0)
    assert e.value.code == rig.RIG_ERR_ZERO_ROW
    # 2 x 3: column 2 is in range (ncols given; unvalidated out-of-range columns are undefined)
    A = rig.CSR(np.array([0, 2, 3]), np.array([0, 1, 2], np.int32), np.array([1.0, np.inf, 3.0]), ncols=3)
    with pytest.raises(rig.RigError) as e:
        rig.rig_build(A, 1, 0.0)
    assert e.value.code == rig.RIG_ERR_NONFINITE
    # a rectangular A with finite values: C = A A^T is 2 x 2 with no off-diagonal entry
    A = rig.CSR(np.array([0, 2, 3]), np.array([0, 1, 2], np.int32), np.array([1.0, 2.0, 3.0]), ncols=3)
    g = rig.rig_build(A, 1, 0.0)
    assert g.n == 2 and g.nnz == 0
    A = rig.CSR(np.array([0, 2, 3]), np.array([1, 0, 2], np.int32), np.array([1.0, 2.0, 3.0]))
    with pytest.raises(rig.RigError) as e:
        rig.rig_build(A, 1, 0.0, rig.RIG_FLAG_VALIDATE)
    assert e.value.code == rig.RIG_ERR_NONCANONICAL
    A = rig.CSR(np.array([0, 2, 3]), np.array([0, 5, 2], np.int32), np.array([1.0, 2.0, 3.0]))
    with pytest.raises(rig.RigError):
        rig.rig_build(A, 1, 0.0, rig.RIG_FLAG_VALIDATE)
    # cutsize: K = 1 -> 0; out-of-range part -> NaN
    w = make_small(1)
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    g = rig.rig_build(A, 1, 0.0)
    assert rig.rig_cutsize(g, torch.zeros(w.n, dtype=torch.int32, device="cuda"), 1).item() == 0.0
    bad = torch.full((w.n,), 4, dtype=torch.int32, device="cuda")
    assert math.isnan(rig.rig_cutsize(g, bad, 4).item())


def test_sym_transpose_path(rig):
    """Pattern-symmetric transpose (a gather) and its fallback, forced on small
    inputs in a fresh process (tests/sym_path_check.py)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RIG_SYM_MIN_NNZ="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "sym_path_check.py")], env=env, cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "sym path ok" in r.stdout


def test_without_row_window(rig):
    """The path without the row-window kernel (what n >= 2^25 rows take; forced
    by RIG_ROWWIN=0 in a fresh process, tests/no_rowwin_check.py): the older
    mid-row passes and the CTA accumulator, graph and cut vs the oracle."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RIG_ROWWIN="0", PYTHONPATH=root)
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "no_rowwin_check.py")], env=env, cwd=root,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "no-rowwin paths ok" in r.stdout


def test_long_rows_and_columns(rig):
    """Mid-row (global far list), huge-row and long-column-sort paths."""
    rng = np.random.default_rng(11)
    n = 20000
    rows, cols = [], []
    # row 0: 3000 distinct columns (f > 2048: the huge-row chain)
    c0 = rng.choice(n, 3000, replace=False); rows += [0] * 3000; cols += list(c0)
    # rows 1..200: 20..600 entries (mid bins: the row-window kernel, global far lists)
    for r in range(1, 201):
        k = int(rng.integers(20, 600))
        cc = rng.choice(n, k, replace=False); rows += [r] * k; cols += list(cc)
    # column 7: 5000 entries (> 4096: in-place global bitonic column sort)
    r7 = rng.choice(np.arange(201, n), 5000, replace=False); rows += list(r7); cols += [7] * 5000
    # column 9: 600 entries (shared-memory column sort)
    r9 = rng.choice(np.arange(201, n), 600, replace=False); rows += list(r9); cols += [9] * 600
    # every row nonempty
    rows += list(range(n)); cols += list(rng.integers(0, n, n))
    rows, cols = np.array(rows), np.array(cols)
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    rp, ci, v = from_triplets(n, n, rows, cols, vals)
    orc = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0)
    A = rig.CSR(rp, ci, v)
    g = rig.rig_build(A, 1, 0.0, rig.RIG_FLAG_DIAG)
    assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc, to_np(g.diag))


@pytest.mark.parametrize("seed", range(3))
def test_mid_rows_deferred(rig, seed):
    """Every row off the merge path (> 8 entries), none huge: rows of 9..40
    random columns overflow the mid kernel's far list (deferred to the huge
    kernel); banded rows with a few far columns do not.  Graph, diag and cut
    against the oracle, with and without drops, and on a shard."""
    rng = np.random.default_rng(500 + seed)
    n = 6000
    rows, cols = [], []
    for r in range(n):
        if r % 7 == 0:  # random columns: every key far from the diagonal
            k = int(rng.integers(9, 40))
            cc = rng.choice(n, k, replace=False)
        else:  # banded, a few far columns
            cc = np.unique(np.concatenate([np.clip(r + rng.integers(-30, 31, 14), 0, n - 1),
                                           rng.integers(0, n, 3)]))
            if cc.size < 9:
                cc = np.unique(np.concatenate([cc, rng.choice(n, 9, replace=False)]))
        rows += [r] * cc.size; cols += list(cc)
    rows, cols = np.array(rows), np.array(cols)
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    rp, ci, v = from_triplets(n, n, rows, cols, vals)
    K = 16
    part = rng.integers(0, K, n).astype(np.int32)
    A = rig.CSR(rp, ci, v)
    for scale, tol in ((1, 0.0), (1, 0.05)):
        orc = oracle.build(rp, ci, v, scale_rows=scale, drop_tol=tol)
        g = rig.rig_build(A, scale, tol, rig.RIG_FLAG_DIAG)
        assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc, to_np(g.diag))
        ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, part, K)[0]
        gc, cut = rig.rig_build_cut(A, torch.as_tensor(part, device="cuda"), K, 0, n, scale, tol)
        assert_graph_equal(to_np(gc.row_ptr), to_np(gc.col_idx), to_np(gc.w), orc)
        assert abs(cut.item() - ocut) <= REL * ocut
    # a shard (local row pointers, global columns)
    a, b = 1234, 4321
    o3 = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0, row_begin=a, row_end=b)
    oc3 = oracle.cutsize(o3.row_ptr, o3.col, o3.w, part, K, row_begin=a)[0]
    g3, cut3 = rig.rig_build_cut(A, torch.as_tensor(part, device="cuda"), K, a, b, 1, 0.0)
    assert_graph_equal(to_np(g3.row_ptr), to_np(g3.col_idx), to_np(g3.w), o3)
    assert abs(cut3.item() - oc3) <= REL * oc3


@pytest.mark.parametrize("seed", range(2))
def test_row_window_path(rig, seed):
    """Row-window path (k_rowwin.cu: every row off the merge path, placed by
    look-back).  Rows of 9..30 random columns keep nearly every product as a
    distinct key, so the graph outgrows the first capacity guess (retry at the
    exact size) and long far lists take the global-scratch redo; a banded
    block exercises the window.  Graph, diag and cut vs the oracle; the cut is
    run-to-run bitwise (per-row sums, fixed tree)."""
    rng = np.random.default_rng(900 + seed)
    n = 5000
    rows, cols = [], []
    for r in range(n):
        if r < n // 2:
            cc = rng.choice(n, int(rng.integers(9, 31)), replace=False)
        else:
            cc = np.unique(np.concatenate([[r], np.clip(r + rng.integers(-60, 61, 20), 0, n - 1),
                                           rng.integers(0, n, 2)]))
        rows += [r] * cc.size; cols += list(cc)
    rows, cols = np.array(rows), np.array(cols)
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    vals[rng.random(rows.size) < 0.2] = 1.0  # equal products: exact cancellations
    vals[rng.random(rows.size) < 0.2] = -1.0
    rp, ci, v = from_triplets(n, n, rows, cols, vals)
    K = 8
    part = rng.integers(0, K, n).astype(np.int32)
    tpart = torch.as_tensor(part, device="cuda")
    A = rig.CSR(rp, ci, v)
    for scale, tol in ((1, 0.0), (0, 0.25)):
        orc = oracle.build(rp, ci, v, scale_rows=scale, drop_tol=tol)
        ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, part, K)[0]
        g = rig.rig_build(A, scale, tol, rig.RIG_FLAG_DIAG)
        assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc, to_np(g.diag))
        cuts = []
        for _ in range(2):
            gc, cut = rig.rig_build_cut(A, tpart, K, 0, n, scale, tol)
            assert_graph_equal(to_np(gc.row_ptr), to_np(gc.col_idx), to_np(gc.w), orc)
            cuts.append(cut.item())
        assert abs(cuts[0] - ocut) <= REL * ocut
        assert cuts[0] == cuts[1]
        plan = rig.Plan(A, scale, tol, rig.RIG_FLAG_DIAG)
        tg = plan.execute()
        assert_graph_equal(to_np(tg.row_ptr), to_np(tg.col_idx), to_np(tg.w), orc, to_np(tg.diag))
        plan.destroy()


@pytest.mark.parametrize("kind", ["rowwin", "merge"])
def test_cut_partition_runs(rig, kind):
    """The fused cut under partitions of every run structure: runs ending at
    4096-row edges, spanning several thousand rows, alternating every row, one
    block for all rows (K = 1, cut 0), a single boundary at the last row, and
    random ids -- the cut vs the oracle on 20000 rows through the row-window
    kernel (banded rows) and the merge kernel (5-point stencil rows)."""
    rng = np.random.default_rng(4242)
    n = 20000
    rows, cols = [], []
    for r in range(n):
        if kind == "rowwin":
            off = rng.choice(np.r_[-40:0, 1:41], 12, replace=False)  # every row > 8 entries
            cc = np.unique(np.concatenate([[r], (r + off) % n, rng.integers(0, n, 2)]))
        else:
            cc = np.unique([(r + d) % n for d in (-100, -1, 0, 1, 100)])
        rows += [r] * cc.size; cols += list(cc)
    rp, ci, v = from_triplets(n, n, np.array(rows), np.array(cols), rng.uniform(-1, 1, len(rows)))
    A = rig.CSR(rp, ci, v)
    orc = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0)
    idx = np.arange(n)
    parts = {
        "chunk_edges": (idx // 4096, 5),
        "long_runs": (idx // 9000, 3),
        "alternate": (idx % 2, 2),
        "one_block": (np.zeros(n, np.int64), 1),
        "last_row": ((idx == n - 1).astype(np.int64), 2),
        "runs_of_7": ((idx // 7) % 4, 4),
        "random": (rng.integers(0, 16, n), 16),
    }
    for name, (pt, K) in parts.items():
        part = pt.astype(np.int32)
        ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, part, K)[0]
        _, cut = rig.rig_build_cut(A, torch.as_tensor(part, device="cuda"), K, 0, n, 1, 0.0)
        assert rig.last_path() == kind, name
        assert abs(cut.item() - ocut) <= REL * max(ocut, 1e-300), name
        if K == 1:
            assert cut.item() == 0.0


@pytest.mark.parametrize("seed", range(2))
def test_long_scattered_rows_cta(rig, seed):
    """Mixed path: short merge rows plus rows of 20..150 scattered columns
    (f_i ~ 100..1500: the row-window kernel in temp mode below 256 products,
    k_row_cta -- CTA per row, shared-memory radix sort -- up to 1280, the
    huge-row chain beyond).  Values with exact ties force cancellations and
    equal-key groups; drops; diag; cut; a shard."""
    rng = np.random.default_rng(77 + seed)
    n = 12000
    rows, cols = [], []
    for r in range(n):
        k = int(rng.integers(20, 150)) if r % 11 == 0 else int(rng.integers(1, 6))
        cc = rng.choice(n, k, replace=False)
        rows += [r] * k; cols += list(cc)
    rows += list(range(n)); cols += list(range(n))
    rows, cols = np.array(rows), np.array(cols)
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    vals[rng.random(rows.size) < 0.25] = 1.0
    vals[rng.random(rows.size) < 0.25] = -1.0
    rp, ci, v = from_triplets(n, n, rows, cols, vals)
    K = 16
    part = rng.integers(0, K, n).astype(np.int32)
    tpart = torch.as_tensor(part, device="cuda")
    A = rig.CSR(rp, ci, v)
    for scale, tol in ((1, 0.0), (0, 0.5)):
        orc = oracle.build(rp, ci, v, scale_rows=scale, drop_tol=tol)
        g = rig.rig_build(A, scale, tol, rig.RIG_FLAG_DIAG)
        assert rig.last_path() == "mixed"
        assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc, to_np(g.diag))
        ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, part, K)[0]
        gc, cut = rig.rig_build_cut(A, tpart, K, 0, n, scale, tol)
        assert_graph_equal(to_np(gc.row_ptr), to_np(gc.col_idx), to_np(gc.w), orc)
        assert abs(cut.item() - ocut) <= REL * ocut
    a, b = 3001, 9002
    o3 = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0, row_begin=a, row_end=b)
    g3 = rig.rig_build_rows(A, a, b, 1, 0.0)
    assert_graph_equal(to_np(g3.row_ptr), to_np(g3.col_idx), to_np(g3.w), o3)


@pytest.mark.parametrize("env", [{}, {"RIG_LONG_SCRATCH_MB": "100"}, {"RIG_LONG_SCRATCH_MB": "1"}])
def test_long_rows_key_ranges(rig, env):
    """Long rows of scattered columns (tests/long_rows_check.py): the CTA
    kernel's key-range launch (crowded buckets split further), a crowded key
    falling to the global far-list / accumulator kernels (scratch allocated
    on demand), a shard.  With RIG_LONG_SCRATCH_MB=100 the longest rows
    exceed the slices and fall back too; with RIG_LONG_SCRATCH_MB=1 there is
    no range launch and every long row takes the fallback chain."""
    if not env:
        import long_rows_check

        long_rows_check.run(0)
        return
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]), **env)
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "long_rows_check.py")], env=e, cwd=root,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "long rows ok" in r.stdout


def test_row_window_early_errors(rig):
    """The row-window path decided before the analysis (every row long):
    device errors raised by the scaling are still reported (read at the final
    synchronisation): a NaN value and an all-zero row."""
    rng = np.random.default_rng(5)
    n = 3000
    rows, cols = [], []
    for r in range(n):  # 12 distinct columns within 20 of the diagonal, + the diagonal
        lo, hi = max(0, r - 20), min(n, r + 21)
        cc = np.unique(np.concatenate([[r], rng.choice(np.arange(lo, hi), 12, replace=False)]))
        rows += [r] * cc.size; cols += list(cc)
    rows, cols = np.array(rows), np.array(cols)
    vals = rng.standard_normal(rows.size)
    rp, ci, v = from_triplets(n, n, rows, cols, vals)
    assert np.diff(rp).min() > 8
    g = rig.rig_build(rig.CSR(rp, ci, v), 1, 0.0)
    assert rig.last_path() == "rowwin"
    orc = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0)
    assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc)
    bad = v.copy()
    bad[17] = np.nan
    with pytest.raises(rig.RigError) as e:
        rig.rig_build(rig.CSR(rp, ci, bad), 1, 0.0)
    assert e.value.code == rig.RIG_ERR_NONFINITE
    z = v.copy()
    z[rp[100]:rp[101]] = 0.0
    with pytest.raises(rig.RigError) as e:
        rig.rig_build(rig.CSR(rp, ci, z), 1, 0.0)
    assert e.value.code == rig.RIG_ERR_ZERO_ROW


def test_mid_row_passes_long_far_lists(rig):
    """Rows of 800..3500 random columns (every key far from the diagonal) run
    through the mid pass, the 768-item far-list pass, the wide window and the
    4096-item global far-list pass (and the huge kernel for the longest);
    short rows take the merge path."""
    rng = np.random.default_rng(4242)
    n = 40000
    rows, cols = [], []
    for r in range(n):
        k = int(rng.integers(800, 3500)) if r % 1500 == 7 else int(rng.integers(1, 4))
        cc = rng.choice(n, k, replace=False)
        rows += [r] * k
        cols += list(cc)
    rows += list(range(n))
    cols += list(range(n))
    rows, cols = np.array(rows), np.array(cols)
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    rp, ci, v = from_triplets(n, n, rows, cols, vals)
    orc = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0)
    g = rig.rig_build(rig.CSR(rp, ci, v), 1, 0.0, rig.RIG_FLAG_DIAG)
    assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc, to_np(g.diag))


@pytest.mark.parametrize("seed", range(4))
def test_random_mixed(rig, seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(500, 3000))
    lens = np.clip(rng.zipf(1.8, n), 1, 300)
    rows = np.repeat(np.arange(n), lens)
    cols = rng.integers(0, n, rows.size)
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    vals[rng.random(rows.size) < 0.3] = 1.0  # exact ties / cancellations
    vals[rng.random(rows.size) < 0.3] = -1.0
    rp, ci, v = from_triplets(n, n, rows, cols, vals)
    for scale, tol in ((1, 0.0), (0, 0.5), (1, 1e-3)):
        orc = oracle.build(rp, ci, v, scale_rows=scale, drop_tol=tol)
        g = rig.rig_build(rig.CSR(rp, ci, v), scale, tol, rig.RIG_FLAG_DIAG)
        assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc, to_np(g.diag))


def test_build_host_e2e(rig):
    w = make_small(2)
    orc = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=1, drop_tol=0.0)
    ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, w.part, w.K)[0]
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    rp, ci, v, part = pin(w.row_ptr), pin(w.col_idx), pin(w.val), pin(w.part)
    orp = torch.empty(w.n + 1, dtype=torch.int64).pin_memory()
    ocol = torch.empty(orc.nnz, dtype=torch.int32).pin_memory()
    ow = torch.empty(orc.nnz, dtype=torch.float64).pin_memory()
    nnz, cut = rig.rig_build_host(rp, ci, v, w.n, 1, 0.0, 0, part, w.K, orp, ocol, ow)
    assert nnz == orc.nnz
    np.testing.assert_array_equal(orp.numpy(), orc.row_ptr)
    np.testing.assert_array_equal(ocol.numpy(), orc.col)
    assert ow.numpy().tobytes() == orc.w.tobytes()
    assert abs(cut - ocut) <= REL * ocut
    small = torch.empty(10, dtype=torch.int32).pin_memory()
    with pytest.raises(rig.RigError):
        rig.rig_build_host(rp, ci, v, w.n, 1, 0.0, 0, part, w.K, orp, small, torch.empty(10, dtype=torch.float64))


# ------------------------------------------------------------------ full size
def _sample_windows(n, rng, k=4, width=1500):
    starts = sorted(set([0, max(0, n - width)] + [int(x) for x in rng.integers(0, n - width, k)]))
    return [(s, min(n, s + width)) for s in starts]


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_full_configs_sampled(rig, cfg):
    """BASELINE.json full sizes in the launch configuration bench.py times
    (rig_build over all rows): totals vs closed forms / oracle products, and
    sampled row windows vs the oracle computing only those rows."""
    w = make(cfg)
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    g = rig.rig_build(A, w.scale_rows, w.drop_tol, rig.RIG_FLAG_DIAG)
    torch.cuda.synchronize()
    closed = {2: 11_980_004, 3: 190_322_400}
    if cfg in closed:
        assert g.nnz == closed[cfg]
    rp = to_np(g.row_ptr)
    rng = np.random.default_rng(cfg)
    a_hat = oracle.scale(w.row_ptr, w.val)[0] if w.scale_rows else w.val
    csc = oracle.transpose(w.n, w.n, w.row_ptr, w.col_idx, a_hat)
    part = torch.as_tensor(w.part, device="cuda")
    for a, b in _sample_windows(w.n, rng):
        o_rp, o_col, o_w, o_diag, _ = oracle.build_from_scaled(w.n, w.n, w.row_ptr, w.col_idx, a_hat, csc,
                                                               w.drop_tol, a, b)
        s, e = int(rp[a]), int(rp[b])
        np.testing.assert_array_equal(rp[a:b + 1] - s, o_rp)
        np.testing.assert_array_equal(to_np(g.col_idx[s:e]), o_col)
        assert to_np(g.w[s:e]).tobytes() == o_w.tobytes()
        assert to_np(g.diag[a:b]).tobytes() == o_diag.tobytes()
        # cutsize of the window: GPU (graph rows a..b) vs oracle
        sub = rig.TensorGraph(g.row_ptr[a:b + 1] - s, g.col_idx[s:e], g.w[s:e], None, a)
        c = rig.rig_cutsize(sub, part, w.K).item()
        oc = oracle.cutsize(o_rp, o_col, o_w, w.part, w.K, row_begin=a)[0]
        assert abs(c - oc) <= REL * max(oc, 1e-300)
    # symmetry spot check via total: sum over j>i equals sum over j<i bitwise-symmetric weights
    assert rig.rig_cutsize(g, torch.zeros(w.n, dtype=torch.int32, device="cuda"), 1).item() == 0.0


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_partition_ip_matrix(rig, cfg):
    """f2: inter-block inner-product matrix and part weights vs the oracle
    (303-309, 1141-1146).  Fixed-point sums: each term is
    truncated at 2^-64 and the total rounded once, so |gpu - oracle| <=
    count * 2^-64 + 4 ulp; the matrix is bitwise symmetric (C is)."""
    w = make_small(cfg)
    orc = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol)
    K = w.K
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    g = rig.rig_build(A, w.scale_rows, w.drop_tol)
    part = torch.as_tensor(w.part, device="cuda")
    for arp in (None, A.row_ptr):
        ip, W = rig.rig_partition_ip(g, part, K, a_row_ptr=arp)
        oip, oW = oracle.ip_matrix(orc.row_ptr, orc.col, orc.w, w.part, K,
                                   a_row_ptr=None if arp is None else w.row_ptr)
        ip = ip.numpy()
        np.testing.assert_array_equal(W.numpy(), oW)
        tol = orc.nnz * 2.0 ** -64 + 8 * 2.0 ** -53 * np.abs(oip)
        assert (np.abs(ip - oip) <= tol).all()
        assert ip.tobytes() == ip.T.copy().tobytes()
        assert np.diag(ip).tolist() == [0.0] * K
    cut = rig.rig_cutsize(g, part, K).item()
    assert abs(np.triu(ip, 1).sum() - cut) <= 1e-12 * cut
    # multi-GPU form: shards accumulate into the same counters (an allreduce)
    split = rig.rig_row_split(A, 3)
    acc = torch.zeros(4 * K * K + 1, dtype=torch.int64, device="cuda")
    Wt = torch.zeros(K, dtype=torch.int64, device="cuda")
    for a, b in zip(split[:-1], split[1:]):
        s = rig.rig_build_rows(A, a, b, w.scale_rows, w.drop_tol)
        rig.rig_partition_ip_accumulate(s, part, K, acc=acc, W=Wt)
    assert rig.rig_partition_ip_finalize(acc, K).numpy().tobytes() == ip.tobytes()
    # bad part id -> error at finalize
    acc2, _ = rig.rig_partition_ip_accumulate(g, torch.full_like(part, K), K)
    with pytest.raises(rig.RigError):
        rig.rig_partition_ip_finalize(acc2, K)


# ---------------------------------------------------------------- f1
def _oracle_sparsified(rp, ci, v, ncols, scale_rows):
    """Oracle pipeline of PAPER.md:572-579: [scale] -> A~ -> graph of A~ A~^T
    (A~ keeps the scaled values, reading R21)."""
    a = oracle.scale(rp, v)[0] if scale_rows else np.asarray(v, dtype=np.float64)
    return oracle.sparsify(rp, ci, a, ncols=ncols)


def _f1_cases():
    from rig_inputs import dense_columns
    cases = []
    for seed, (n, per, nd, dn, lv, sc) in enumerate([
            (3000, 5, 4, 700, 0, 1),     # scaled, distinct magnitudes
            (2500, 4, 3, 900, 2, 0),     # unscaled, many |value| ties
            (1200, 3, 2, 1100, 1, 0),    # all |values| equal: ties span many chunks
            (5000, 6, 8, 60, 0, 1),      # dense columns just above T = 71? (no: 60 < 71) -> identity
            (4099, 5, 5, 2000, 0, 1)]):  # ragged sizes
        rng = np.random.default_rng(900 + seed)
        rp, ci, v = dense_columns(n, rng, per_row=per, n_dense=nd, dense_nnz=dn, levels=lv)
        cases.append((f"dense{seed}", n, rp, ci, v, sc))
    # the paper's 25 x 25 example
    D = np.eye(25)
    for r in range(25):
        if r not in (2, 19):
            D[r, 11] = 1.0 + r / 7.0
    rp, ci, v = from_dense(D)
    cases.append(("paper25", 25, rp, ci, v, 1))
    w = make_small(2)
    cases.append(("stencil", w.n, w.row_ptr, w.col_idx, w.val, 1))
    return cases


@pytest.mark.parametrize("case", _f1_cases(), ids=lambda c: c[0])
def test_sparsify_bitexact(rig, case):
    name, n, rp, ci, v, sc = case
    trp, tci, tv = _oracle_sparsified(rp, ci, v, n, sc)
    A = rig.CSR(rp, ci, v, ncols=n)
    At = rig.rig_sparsify(A, sc)
    np.testing.assert_array_equal(to_np(At.row_ptr), trp)
    np.testing.assert_array_equal(to_np(At.col_idx), tci)
    assert to_np(At.val).tobytes() == tv.tobytes()


@pytest.mark.parametrize("case", _f1_cases(), ids=lambda c: c[0])
def test_sparsified_graph_bitexact(rig, case):
    """G~_RIP (RIG_FLAG_SPARSIFY) == oracle graph of A~ A~^T; shards and the
    staged API agree."""
    name, n, rp, ci, v, sc = case
    trp, tci, tv = _oracle_sparsified(rp, ci, v, n, sc)
    orc = oracle.build(trp, tci, tv, ncols=n, scale_rows=0, drop_tol=0.0)
    A = rig.CSR(rp, ci, v, ncols=n)
    flags = rig.RIG_FLAG_DIAG | rig.RIG_FLAG_SPARSIFY
    g = rig.rig_build(A, sc, 0.0, flags)
    assert g.nnz == orc.nnz
    assert_graph_equal(to_np(g.row_ptr), to_np(g.col_idx), to_np(g.w), orc, to_np(g.diag))
    plan = rig.Plan(A, sc, 0.0, flags)
    tg = plan.execute()
    assert_graph_equal(to_np(tg.row_ptr), to_np(tg.col_idx), to_np(tg.w), orc, to_np(tg.diag))
    plan.destroy()
    split = rig.rig_row_split(A, 3)
    cols, ws = [], []
    for a, b in zip(split[:-1], split[1:]):
        s = rig.rig_build_rows(A, a, b, sc, 0.0, flags)
        cols.append(to_np(s.col_idx))
        ws.append(to_np(s.w))
    np.testing.assert_array_equal(np.concatenate(cols), orc.col)
    assert np.concatenate(ws).tobytes() == orc.w.tobytes()


def test_sparsify_large_bitexact(rig):
    """Full-size f1 case: n = 1M rows, 8 dense columns of 60k rows (T = 1000),
    A~ and the graph of A~ A~^T bit-exact."""
    from rig_inputs import dense_columns
    n = 1_000_000
    rp, ci, v = dense_columns(n, np.random.default_rng(77), per_row=5, n_dense=8, dense_nnz=60_000)
    trp, tci, tv = _oracle_sparsified(rp, ci, v, n, 1)
    A = rig.CSR(rp, ci, v, ncols=n)
    At = rig.rig_sparsify(A, 1)
    np.testing.assert_array_equal(to_np(At.row_ptr), trp)
    np.testing.assert_array_equal(to_np(At.col_idx), tci)
    assert to_np(At.val).tobytes() == tv.tobytes()
    orc = oracle.build(trp, tci, tv, ncols=n, scale_rows=0)
    g = rig.rig_build(A, 1, 0.0, rig.RIG_FLAG_SPARSIFY)
    np.testing.assert_array_equal(to_np(g.row_ptr), orc.row_ptr)
    np.testing.assert_array_equal(to_np(g.col_idx), orc.col)
    assert to_np(g.w).tobytes() == orc.w.tobytes()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_int_weights_exact(rig, cfg):
    """wgt = ceil(alpha * w) equals the oracle's exact integer
    computation for every edge; scaled configs land in [1, alpha]."""
    w = make_small(cfg)
    orc = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol)
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    g = rig.rig_build(A, w.scale_rows, w.drop_tol)
    for alpha in (1, 10_000, 2 ** 31 - 1, 2 ** 53):
        got = to_np(rig.rig_int_weights(g.w, alpha))
        np.testing.assert_array_equal(got, oracle.int_weights(orc.w, alpha))
        if w.scale_rows and got.size:
            assert got.min() >= 1 and got.max() <= alpha


def test_int_weights_edge_values(rig):
    rng = np.random.default_rng(3)
    x = np.r_[rng.random(5000), rng.random(500) * 1e-12, 0.1, 0.3, 0.7, 1.0, 0.5, 2.0 ** -60, 5e-324, 0.0,
              np.nextafter(1.0, 0.0), np.nextafter(0.1, 1.0), 3.0, 300.0]
    xt = torch.as_tensor(x, device="cuda")
    for alpha in (1, 3, 10_000, 2 ** 31 - 1, 2 ** 53):
        np.testing.assert_array_equal(to_np(rig.rig_int_weights(xt, alpha)), oracle.int_weights(x, alpha))
    bad = torch.tensor([-0.5, float("inf"), float("nan"), 1e300], dtype=torch.float64, device="cuda")
    assert to_np(rig.rig_int_weights(bad, 10)).tolist() == [-1, -1, -1, -1]
    with pytest.raises(rig.RigError):
        rig.rig_int_weights(xt, 0)


# ------------------------------------------------------------------ f4
def _sym_int_graph(n, edges):
    r, c, w = [], [], []
    for u, v, x in edges:
        r += [u, v]
        c += [v, u]
        w += [x, x]
    rp, ci, vv = from_triplets(n, n, np.array(r), np.array(c), np.array(w, dtype=np.float64))
    return rp, ci, vv.astype(np.int64)


def _check_f4(rig, rp, ci, wg, vw=None, rounds=4):
    from oracle.coarsen import coarsen, hem_match

    m_o = hem_match(rp, ci, wg, rounds=rounds)
    dev = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    m_g = rig.rig_hem_match(dev(rp), dev(ci), dev(wg), rounds=rounds)
    np.testing.assert_array_equal(to_np(m_g), m_o)
    cmap, nc, crp, cci, cw, cvw = coarsen(rp, ci, wg, m_o, vwgt=vw)
    out = rig.rig_coarsen(dev(rp), dev(ci), dev(wg), m_g, vwgt=None if vw is None else dev(vw))
    assert out["n"] == nc and out["nnz"] == cci.size
    np.testing.assert_array_equal(to_np(out["cmap"]), cmap)
    np.testing.assert_array_equal(to_np(out["row_ptr"]), crp)
    np.testing.assert_array_equal(to_np(out["col_idx"]), cci)
    np.testing.assert_array_equal(to_np(out["wgt"]), cw)
    np.testing.assert_array_equal(to_np(out["vwgt"]), cvw)


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_f4_matching_and_coarsening_on_grip(rig, cfg):
    """Heavy-edge matching and one coarsening step of G_RIP with the METIS
    weights ceil(1e4 * cost): device == oracle, exactly."""
    w = make_small(cfg)
    A, g = gpu_build(rig, w, flags=0)
    wg = rig.rig_int_weights(g.w, 10_000)
    vw = np.diff(w.row_ptr).astype(np.int64)  # vertex weight: nnz of the row
    _check_f4(rig, to_np(g.row_ptr), to_np(g.col_idx), to_np(wg), vw=vw)


@pytest.mark.parametrize("seed", range(3))
def test_f4_random_ties_and_big_rows(rig, seed):
    """Small integer weights (many ties, smallest-index rule), isolated
    vertices, and a hub of 1500 neighbours (coarse rows beyond 1024 items take
    the global-scratch sort)."""
    rng = np.random.default_rng(77 + seed)
    n = 3000
    edges = {}
    for _ in range(9000):
        u, v = map(int, rng.integers(0, n - 50, 2))  # the last 50 vertices stay isolated
        if u != v:
            edges[(min(u, v), max(u, v))] = int(rng.integers(1, 4))
    hub = int(rng.integers(0, n - 50))
    for v in rng.choice(n - 50, 1500, replace=False):
        if int(v) != hub:
            edges[(min(hub, int(v)), max(hub, int(v)))] = int(rng.integers(1, 4))
    rp, ci, wg = _sym_int_graph(n, [(u, v, x) for (u, v), x in edges.items()])
    _check_f4(rig, rp, ci, wg, rounds=1 + seed * 3)
