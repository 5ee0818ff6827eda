"""Pins the CPU oracle to things other than itself (CPU-only, `-m "not gpu"`).

Each pin is chosen so a plausible oracle mistake (dropped term, wrong sign or
index, transposed operand, wrong rounding/order, wrong drop rule) fails one:

  * paper values: c_24 = 216, nnz(AA^T) = 531,
    SPEC.md:142 scaling (3,4)->(0.6,0.8)                       [tests/golden/]
  * exact integer arithmetic: small-integer A gives C = A A^T exactly, so the
    oracle must equal numpy's int64 product entry for entry, and the graph must
    be the off-diagonal nonzero pattern (edge iff r_i r_j^T != 0)
  * an exact-rational model of the ordering contract (DESIGN.md §3 R4): each
    c_ij recomputed pairwise by a sorted-intersection merge with
    correctly-rounded fma via fractions.Fraction -> bitwise equality
  * dense BLAS A_hat A_hat^T within the forward-error bound gamma_m sum|a a|
  * library routines for sub-steps: scipy CSR->CSC, scipy boolean product
  * closed forms (stencil nnz(C), products) and invariants (bitwise symmetry,
    diag = squared row norms / 1, Cauchy-Schwarz)
  * cutsize: math.fsum over the cut edges, cut = total - intra, K=1 -> 0, all
    parts distinct -> total, block-diagonal -> 0, brute-force interIP from
    dense row inner products (eq. ip_km)
  * f1 sparsification: the paper's 25x25 dense-column example keeps 5 entries
    (PAPER.md:567-577); the kept set equals a brute-force rank count per entry
    (#entries of its column that beat it < T); T = ceil(sqrt(n)) against
    math.isqrt; no dense column -> A~ = A; ties -> lowest rows
  * f1 integer weights: exact ceil(alpha * w) by fractions.Fraction, and the
    paper's range [1, alpha] for costs in (0, 1]
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from rig_inputs import dense_columns, from_dense, from_triplets, make, make_small, part_contiguous, stencil2d, stencil3d
from rig_testutil import read_golden

U = 2.0 ** -53


def exact_fma(a, b, c):
    # float(Fraction) is int/int true division: correctly rounded in CPython
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def rand_csr(n, m, density, rng, ints=False):
    D = (rng.random((n, m)) < density).astype(np.float64)
    if ints:
        D *= rng.integers(-3, 4, size=(n, m))
    else:
        D *= rng.standard_normal((n, m))
    for i in range(n):  # no empty rows
        if not D[i].any():
            D[i, rng.integers(0, m)] = 1.0 if ints else 1.0 + rng.random()
    return D, from_dense(D)


def dense_graph(g, n):
    G = np.zeros((g.row_ptr.size - 1, n))
    for r in range(g.row_ptr.size - 1):
        s, e = g.row_ptr[r], g.row_ptr[r + 1]
        G[r, g.col[s:e]] = g.w[s:e]
    return G


# ---------------------------------------------------------------- paper values
def test_paper_216_edge_cost():
    lines = read_golden("paper_216.txt")
    n = int(lines[0][1])
    trip = [(int(a) - 1, int(b) - 1, float(c)) for a, b, c in (l for l in lines[1:] if l[0] != "expect")]
    rp, ci, v = from_triplets(n, n, [t[0] for t in trip], [t[1] for t in trip], [t[2] for t in trip])
    g = oracle.build(rp, ci, v, scale_rows=0, drop_tol=0.0)
    G = dense_graph(g, n)
    for l in (l for l in lines if l[0] == "expect"):
        i, j, want = int(l[1]) - 1, int(l[2]) - 1, float(l[3])
        assert G[i, j] == want


def test_paper_531_dense_column():
    kv = {l[0]: l[1:] for l in read_golden("paper_531.txt")}
    n = int(kv["n"][0])
    dc = int(kv["dense_col"][0]) - 1
    out = {int(x) - 1 for x in kv["rows_not_in_dense_col"]}
    D = np.eye(n)
    for r in range(n):
        if r not in out:
            D[r, dc] = 1.0 + r / 7.0
    assert np.count_nonzero(D[:, dc]) == 23
    rp, ci, v = from_dense(D)
    g = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0)
    assert int(g.nnzc.sum()) == int(kv["expect_nnz_C"][0])
    assert g.nnz == int(kv["expect_graph_nnz_directed"][0])
    assert g.nnz // 2 == int(kv["expect_undirected_edges"][0])


def test_spec_scaling_345_bitwise():
    lines = read_golden("spec_scaling_345.txt")
    row = [float(x) for x in lines[0][1:]]
    want = [float(x) for x in lines[1][1:]]
    out, norms = oracle.scale(np.array([0, 2]), np.array(row))
    assert out.tolist() == want and norms[0] == 5.0


# ---------------------------------------------------- exact integer arithmetic
@pytest.mark.parametrize("seed", range(6))
def test_integer_matrix_exact_product_and_pattern(seed):
    rng = np.random.default_rng(seed)
    n, m = 120, 90
    D, (rp, ci, v) = rand_csr(n, m, 0.06, rng, ints=True)
    # force exact cancellations: rows 0,1 = (1,1,0..) and (1,-1,0..) -> c_01 = 0
    D[0, :] = 0; D[1, :] = 0
    D[0, 5] = 1; D[0, 6] = 1; D[1, 5] = 1; D[1, 6] = -1
    rp, ci, v = from_dense(D)
    Di = D.astype(np.int64)
    C = Di @ Di.T
    g = oracle.build(rp, ci, v, ncols=m, scale_rows=0, drop_tol=0.0)
    G = dense_graph(g, n)
    off = ~np.eye(n, dtype=bool)
    want = np.where(off, np.abs(C), 0).astype(np.float64)
    np.testing.assert_array_equal(G, want)
    assert G[0, 1] == 0.0  # exact cancellation -> no edge
    np.testing.assert_array_equal(g.diag, np.diag(C).astype(np.float64))
    # structural nnz of C (incl. diagonal) = boolean pattern product (library)
    P = sp.csr_matrix((np.ones_like(v), ci, rp), shape=(n, m))
    pat = (P @ P.T).tocsr()
    np.testing.assert_array_equal(g.nnzc, np.diff(pat.indptr))
    # ascending columns within every row
    for r in range(n):
        s, e = g.row_ptr[r], g.row_ptr[r + 1]
        assert np.all(np.diff(g.col[s:e]) > 0)


# ---------------------------------------- exact-rational ordering-contract model
def model_scale(rp, v):
    out = np.empty_like(v)
    for i in range(rp.size - 1):
        ss = 0.0
        for p in range(rp[i], rp[i + 1]):
            ss = exact_fma(v[p], v[p], ss)
        nrm = math.sqrt(ss)
        for p in range(rp[i], rp[i + 1]):
            out[p] = v[p] / nrm
    return out


def model_c(rp, ci, vh, i, j):
    """Pairwise sorted-intersection merge, ascending k, exact-rational fma."""
    a, b = rp[i], rp[j]
    ea, eb = rp[i + 1], rp[j + 1]
    acc, hit = 0.0, False
    while a < ea and b < eb:
        if ci[a] == ci[b]:
            acc = exact_fma(vh[a], vh[b], acc)
            hit = True
            a += 1; b += 1
        elif ci[a] < ci[b]:
            a += 1
        else:
            b += 1
    return hit, acc


@pytest.mark.parametrize("seed,scale", [(0, 1), (1, 1), (2, 0), (3, 1)])
def test_ordering_contract_exact_rational_model(seed, scale):
    rng = np.random.default_rng(100 + seed)
    n = 70
    D, (rp, ci, v) = rand_csr(n, n, 0.08, rng)
    D[3] = D[9]  # a duplicate row: c_{3,9} = c_{3,3}
    rp, ci, v = from_dense(D)
    vh = model_scale(rp, v) if scale else v
    g = oracle.build(rp, ci, v, scale_rows=scale, drop_tol=0.0, keep_intermediates=True)
    if scale:
        assert g.a_hat.tobytes() == vh.tobytes()
    for i in range(n):
        cols, ws = [], []
        for j in range(n):
            hit, c = model_c(rp, ci, vh, i, j)
            if j == i:
                assert hit and g.diag[i] == c
            elif hit and abs(c) > 0.0:
                cols.append(j); ws.append(abs(c))
        s, e = g.row_ptr[i], g.row_ptr[i + 1]
        assert g.col[s:e].tolist() == cols
        assert g.w[s:e].tobytes() == np.array(ws, dtype=np.float64).tobytes()
    Gd = dense_graph(g, n)
    # identical rows, identical chains: c_{3,9} == c_{3,3} bitwise
    assert Gd[3, 9] == g.diag[3]


# ------------------------------------------------------------- dense BLAS bound
def test_tiny_config_vs_dense_blas():
    w = make(1)
    g = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=1, drop_tol=0.0, keep_intermediates=True)
    n = w.n
    Ah = sp.csr_matrix((g.a_hat, w.col_idx, w.row_ptr), shape=(n, n)).toarray()
    C = Ah @ Ah.T
    absC = np.abs(Ah) @ np.abs(Ah).T
    cnt = (Ah != 0).astype(np.float64) @ (Ah != 0).astype(np.float64).T
    gam = cnt * U / (1 - cnt * U)
    G = dense_graph(g, n)
    off = ~np.eye(n, dtype=bool)
    struct = cnt > 0
    # every structural off-diagonal entry is an edge (no exact zeros with N(0,1))
    assert np.array_equal(G > 0, struct & off)
    err = np.abs(G - np.abs(C))[struct & off]
    assert np.all(err <= 2 * gam[struct & off] * absC[struct & off] + 1e-300)
    np.testing.assert_allclose(g.diag, np.diag(C), rtol=0, atol=8 * U * 6)


# --------------------------------------------------------- library sub-steps
def test_transpose_matches_scipy_and_products():
    w = make_small(4)
    cp, ri, vt = oracle.transpose(w.n, w.n, w.row_ptr, w.col_idx, w.val)
    A = sp.csr_matrix((w.val, w.col_idx, w.row_ptr), shape=(w.n, w.n)).tocsc()
    A.sort_indices()
    np.testing.assert_array_equal(cp, A.indptr)
    np.testing.assert_array_equal(ri, A.indices)
    assert vt.tobytes() == A.data.tobytes()
    f, total = oracle.row_products(w.row_ptr, w.col_idx, cp)
    collen = np.bincount(w.col_idx, minlength=w.n).astype(np.int64)
    assert total == int((collen ** 2).sum())
    np.testing.assert_array_equal(f, np.add.reduceat(collen[w.col_idx], w.row_ptr[:-1])
                                  * (np.diff(w.row_ptr) > 0))


# ----------------------------------------------------------------- closed forms
def nnzc_2d(N):
    return N * N + 4 * N * (N - 1) + 4 * N * (N - 2) + 4 * (N - 1) ** 2


def nnzc_3d(N):
    return N ** 3 + 6 * N * N * (N - 1) + 6 * N * N * (N - 2) + 12 * N * (N - 1) ** 2


@pytest.mark.parametrize("N", [5, 9, 31])
def test_stencil_closed_forms(N):
    rng = np.random.default_rng(N)
    for gen, nnzc in ((stencil2d, nnzc_2d), (stencil3d, nnzc_3d)):
        if gen is stencil3d and N > 9:
            continue
        rp, ci, v = gen(N, rng)
        g = oracle.build(rp, ci, v, scale_rows=1, drop_tol=0.0)
        n = rp.size - 1
        assert int(g.nnzc.sum()) == nnzc(N)
        assert g.nnz == nnzc(N) - n  # no drops: same-sign products, no cancellation
        P = sp.csr_matrix((np.ones_like(v), ci, rp), shape=(n, n))
        collen = np.diff(P.tocsc().indptr)
        assert g.products == int((collen.astype(np.int64) ** 2).sum())
    # values printed in SURVEY.md §8(c) c3 for the full configs
    assert nnzc_2d(1000) == 12_980_004 and nnzc_3d(200) == 198_322_400


def test_config2_full_counts():
    w = make(2)
    g = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=1, drop_tol=0.0)
    assert g.products == 24_964_008
    assert int(g.nnzc.sum()) == 12_980_004
    assert g.nnz == 11_980_004


# ------------------------------------------------------------------ invariants
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6, 7])
def test_invariants_small_configs(cfg):
    w = make_small(cfg)
    g = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol,
                     keep_intermediates=True)
    n = w.n
    # bitwise symmetry of structure and weights (ordering contract consequence)
    M = sp.csr_matrix((g.w, g.col, g.row_ptr), shape=(n, n))
    MT = M.T.tocsr(); MT.sort_indices()
    np.testing.assert_array_equal(M.indptr, MT.indptr)
    np.testing.assert_array_equal(M.indices, MT.indices)
    assert M.data.tobytes() == MT.data.tobytes()
    assert np.all(g.col != np.repeat(np.arange(n), np.diff(g.row_ptr)))  # no self loops
    assert np.all(g.w > w.drop_tol)
    lens = np.diff(w.row_ptr)
    if w.scale_rows:
        # diag(C) = squared norms of unit rows = 1 within (nnz_i + 3) u
        assert np.all(np.abs(g.diag - 1.0) <= (lens + 3) * U)
        # Cauchy-Schwarz |c_ij| <= 1 (+ rounding)
        assert g.w.max() <= 1.0 + (lens.max() + 3) * U
    else:
        ss = np.array([math.fsum(x * x for x in w.val[w.row_ptr[i]:w.row_ptr[i + 1]]) for i in range(n)])
        np.testing.assert_allclose(g.diag, ss, rtol=(lens.max() + 2) * U)


# ---------------------------------------------------------------- edge cases
def test_zero_row_and_nonfinite_errors():
    rp = np.array([0, 2, 2, 3]); ci = np.array([0, 1, 2], np.int32); v = np.array([1.0, 2.0, 3.0])
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(rp, ci, v, scale_rows=1)
    assert e.value.code == oracle.ORC_ERR_ZERO_ROW
    g = oracle.build(rp, ci, v, scale_rows=0)  # unscaled: empty row = isolated vertex
    assert g.row_ptr.tolist() == [0, 0, 0, 0] and g.nnzc.tolist() == [1, 0, 1]
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(rp, ci, np.array([1.0, np.nan, 3.0]), scale_rows=1)
    assert e.value.code == oracle.ORC_ERR_NONFINITE


def test_degenerate_shapes():
    g = oracle.build(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0), scale_rows=0)
    assert g.nnz == 0 and g.row_ptr.tolist() == [0]
    g = oracle.build(np.array([0, 3]), np.array([0, 4, 7], np.int32), np.array([1., 2., 3.]), ncols=9, scale_rows=1)
    assert g.nnz == 0 and abs(g.diag[0] - 1.0) <= 4 * U
    # drop rule is strict: |c| == drop_tol is dropped, just below is kept
    D = np.array([[1.0, 0.0], [0.5, 1.0]])
    rp, ci, v = from_dense(D)
    assert oracle.build(rp, ci, v, scale_rows=0, drop_tol=0.5).nnz == 0
    assert oracle.build(rp, ci, v, scale_rows=0, drop_tol=np.nextafter(0.5, 0)).nnz == 2
    # duplicate rows: off-diagonal cost equals the diagonal
    D = np.array([[1.0, 2.0, 0.0], [1.0, 2.0, 0.0], [0.0, 0.0, 3.0]])
    rp, ci, v = from_dense(D)
    g = oracle.build(rp, ci, v, scale_rows=0)
    assert dense_graph(g, 3)[0, 1] == g.diag[0] == 5.0


# ---------------------------------------------------------------- cutsize
def test_cutsize_pins_tiny():
    w = make(1)
    g = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=1, drop_tol=0.0, keep_intermediates=True)
    n = w.n
    cut, total, intra = oracle.cutsize(g.row_ptr, g.col, g.w, w.part, w.K)
    rows = np.repeat(np.arange(n), np.diff(g.row_ptr))
    sel = (g.col > rows) & (w.part[rows] != w.part[g.col])
    exact = math.fsum(g.w[sel])
    assert abs(cut - exact) <= 2 * U * exact
    assert abs(total - math.fsum(g.w[g.col > rows])) <= 2 * U * total
    assert abs(cut - (total - intra)) <= 4 * U * total
    # brute-force interIP = sum_{k<m} ip_km from dense row inner products
    Ah = sp.csr_matrix((g.a_hat, w.col_idx, w.row_ptr), shape=(n, n)).toarray()
    C = np.abs(Ah @ Ah.T)
    ip = np.zeros((w.K, w.K))
    for k in range(w.K):
        for m in range(w.K):
            ip[k, m] = C[np.ix_(w.part == k, w.part == m)].sum()
    inter = sum(ip[k, m] for k in range(w.K) for m in range(k + 1, w.K))
    assert abs(cut - inter) <= 1e-12 * inter
    # K = 1 -> 0 exactly; all distinct -> total
    assert oracle.cutsize(g.row_ptr, g.col, g.w, np.zeros(n, np.int32), 1)[0] == 0.0
    assert oracle.cutsize(g.row_ptr, g.col, g.w, np.arange(n, dtype=np.int32), n)[0] == total
    with pytest.raises(oracle.OracleError):
        oracle.cutsize(g.row_ptr, g.col, g.w, np.full(n, 4, np.int32), 4)


def test_cutsize_block_diagonal_zero():
    rng = np.random.default_rng(7)
    D1, _ = rand_csr(40, 40, 0.1, rng)
    D2, _ = rand_csr(30, 30, 0.1, rng)
    D = np.zeros((70, 70)); D[:40, :40] = D1; D[40:, 40:] = D2
    rp, ci, v = from_dense(D)
    g = oracle.build(rp, ci, v, scale_rows=1)
    part = np.r_[np.zeros(40, np.int32), np.ones(30, np.int32)]
    cut, total, intra = oracle.cutsize(g.row_ptr, g.col, g.w, part, 2)
    assert cut == 0.0 and total == intra > 0


def test_shard_concatenation_equals_full():
    w = make_small(5)
    full = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=0, drop_tol=w.drop_tol)
    cuts = []
    split = [0, 7001, 19000, w.n]
    cols, ws = [], []
    for a, b in zip(split[:-1], split[1:]):
        s = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=0, drop_tol=w.drop_tol, row_begin=a, row_end=b)
        cols.append(s.col); ws.append(s.w)
        cuts.append(oracle.cutsize(s.row_ptr, s.col, s.w, w.part, w.K, row_begin=a)[0])
    np.testing.assert_array_equal(np.concatenate(cols), full.col)
    assert np.concatenate(ws).tobytes() == full.w.tobytes()
    c_full = oracle.cutsize(full.row_ptr, full.col, full.w, w.part, w.K)[0]
    assert abs(sum(cuts) - c_full) <= 1e-12 * c_full


def test_uniform_partition_sizes_golden():
    for l in read_golden("spec_uniform_partition.txt"):
        n, K = int(l[0]), int(l[1])
        sizes = np.bincount(part_contiguous(n, K), minlength=K).tolist()
        assert sizes == [int(x) for x in l[2:]]


def test_ip_matrix_pins():
    """f2: the oracle's inter-block inner-product matrix
    (eq. ip_km) against exact per-cell sums of the graph,
    brute-force dense row inner products, sum_{k<m} ip_km = cutsize
    (PAPER.md:519-529), symmetry, and the part weights (eq16,
    1141-1146 eq. Wk)."""
    w = make(1)
    g = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=1, drop_tol=0.0, keep_intermediates=True)
    n, K = w.n, w.K
    ip, W = oracle.ip_matrix(g.row_ptr, g.col, g.w, w.part, K)
    rows = np.repeat(np.arange(n), np.diff(g.row_ptr))
    pk, pm = w.part[rows], w.part[g.col]
    for k in range(K):
        assert ip[k, k] == 0.0
        for m in range(K):
            if m != k:
                exact = math.fsum(g.w[(pk == k) & (pm == m)])
                assert abs(ip[k, m] - exact) <= 2 * U * exact
    assert np.allclose(ip, ip.T, rtol=4 * U, atol=0)
    cut = oracle.cutsize(g.row_ptr, g.col, g.w, w.part, K)[0]
    assert abs(np.triu(ip, 1).sum() - cut) <= 1e-13 * cut
    # brute force from dense A_hat A_hat^T (independent of the graph build)
    Ah = sp.csr_matrix((g.a_hat, w.col_idx, w.row_ptr), shape=(n, n)).toarray()
    C = np.abs(Ah @ Ah.T)
    for k in range(K):
        for m in range(K):
            if m != k:
                ref = C[np.ix_(w.part == k, w.part == m)].sum()
                assert abs(ip[k, m] - ref) <= 1e-12 * ref
    # part weights: unit and nnz(r_i)
    np.testing.assert_array_equal(W, np.bincount(w.part, minlength=K))
    _, Wn = oracle.ip_matrix(g.row_ptr, g.col, g.w, w.part, K, a_row_ptr=w.row_ptr)
    np.testing.assert_array_equal(Wn, np.bincount(w.part, weights=np.diff(w.row_ptr), minlength=K).astype(np.int64))
    assert Wn.sum() == w.nnz
    # K = 1: nothing is inter-block
    ip1, W1 = oracle.ip_matrix(g.row_ptr, g.col, g.w, np.zeros(n, np.int32), 1)
    assert ip1[0, 0] == 0.0 and W1[0] == n
    with pytest.raises(oracle.OracleError):
        oracle.ip_matrix(g.row_ptr, g.col, g.w, np.full(n, K, np.int32), K)


def test_ip_matrix_block_diagonal_zero():
    rng = np.random.default_rng(9)
    D1, _ = rand_csr(30, 30, 0.15, rng)
    D2, _ = rand_csr(25, 25, 0.15, rng)
    D = np.zeros((55, 55)); D[:30, :30] = D1; D[30:, 30:] = D2
    rp, ci, v = from_dense(D)
    g = oracle.build(rp, ci, v, scale_rows=1)
    part = np.r_[np.zeros(30, np.int32), np.ones(25, np.int32)]
    ip, W = oracle.ip_matrix(g.row_ptr, g.col, g.w, part, 2)
    assert not ip.any() and W.tolist() == [30, 25]


# ---------------------------------------------------------------- f1
def test_dense_threshold_is_ceil_sqrt():
    for n in list(range(0, 200)) + [10**6, 4_000_000, 4_000_001, (1 << 31) - 1]:
        t = oracle.dense_threshold(n)
        assert t == (math.isqrt(n - 1) + 1 if n > 0 else 0)


def brute_kept(rp, ci, v, T):
    """Entry (i, k) survives iff fewer than T entries of column k beat it
    (larger |value|, or equal |value| and a lower row)."""
    n = rp.size - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    keep = np.ones(ci.size, bool)
    for p in range(ci.size):
        same = ci == ci[p]
        if same.sum() <= T:
            continue
        a = np.abs(v)
        beats = same & ((a > a[p]) | ((a == a[p]) & (rows < rows[p])))
        keep[p] = beats.sum() < T
    return keep


def test_sparsify_paper_25x25_example():
    kv = {l[0]: l[1:] for l in read_golden("paper_531.txt")}
    n = int(kv["n"][0])
    dc = int(kv["dense_col"][0]) - 1
    out = {int(x) - 1 for x in kv["rows_not_in_dense_col"]}
    D = np.eye(n)
    for r in range(n):
        if r not in out:
            D[r, dc] = 1.0 + r / 7.0
    rp, ci, v = from_dense(D)
    ahat, _ = oracle.scale(rp, v)
    trp, tci, tv = oracle.sparsify(rp, ci, ahat)
    # "keeping 5 largest nonzeros in the dense column"
    assert np.count_nonzero(tci == dc) == 5
    for k in range(n):
        if k != dc:
            assert np.count_nonzero(tci == k) == np.count_nonzero(ci == k)
    # row dc holds only its dense-column entry (|a_hat| = 1, the largest), the
    # other rows' |a_hat| = d / sqrt(1 + d^2) grows with d = 1 + r/7
    kept_rows = sorted(np.repeat(np.arange(n), np.diff(trp))[tci == dc].tolist())
    assert kept_rows == [dc, 21, 22, 23, 24]
    # C~ = A~ A~^T: a 5-clique plus the other 20 diagonals -> 45 (vs 531)
    g = oracle.build(trp, tci, tv, scale_rows=0)
    assert int(g.nnzc.sum()) == 45 and g.nnz == 20


@pytest.mark.parametrize("seed,levels", [(0, 0), (1, 0), (2, 2), (3, 1)])
def test_sparsify_brute_force_rank(seed, levels):
    rng = np.random.default_rng(700 + seed)
    n = 60 + 7 * seed
    rp, ci, v = dense_columns(n, rng, per_row=3, n_dense=3, dense_nnz=n // 3, levels=levels)
    T = oracle.dense_threshold(n)
    keep = brute_kept(rp, ci, v, T)
    trp, tci, tv = oracle.sparsify(rp, ci, v)
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.array_equal(trp, np.r_[0, np.cumsum(np.bincount(rows[keep], minlength=n))])
    assert np.array_equal(tci, ci[keep]) and np.array_equal(tv, v[keep])
    assert np.bincount(tci, minlength=n).max() <= T


def test_sparsify_ties_take_lowest_rows():
    n = 16  # T = 4
    rows = np.arange(n)
    rp, ci, v = from_triplets(n, 40, np.r_[rows, rows], np.r_[np.full(n, 3), rows + 8],
                              np.r_[np.full(n, -2.0), np.ones(n)])
    trp, tci, tv = oracle.sparsify(rp, ci, v, ncols=40)
    kept = np.repeat(np.arange(n), np.diff(trp))[tci == 3]
    assert kept.tolist() == [0, 1, 2, 3]
    # columns 8..23 hold one entry each: unchanged
    assert np.count_nonzero(tci != 3) == n


def test_sparsify_no_dense_column_is_identity():
    w = make_small(2)  # 5-point stencil: column counts <= 5 <= ceil(sqrt(n))
    trp, tci, tv = oracle.sparsify(w.row_ptr, w.col_idx, w.val)
    assert np.array_equal(trp, w.row_ptr) and np.array_equal(tci, w.col_idx) and np.array_equal(tv, w.val)


def test_int_weights_exact_ceiling():
    rng = np.random.default_rng(5)
    w = np.r_[rng.random(2000), rng.random(200) * 1e-9, 0.1, 0.3, 1.0, 0.5, 2.0 ** -60,
              np.nextafter(1.0, 0.0), 5e-324, 0.0]
    for alpha in (1, 3, 10_000, 2 ** 31 - 1, 2 ** 53):
        got = oracle.int_weights(w, alpha)
        want = [math.ceil(Fraction(alpha) * Fraction(float(x))) for x in w]
        assert got.tolist() == want
    # 0.1 is slightly above 1/10, so ceil(10^4 * 0.1) = 1001 (1000 in naive fp)
    assert oracle.int_weights(np.array([0.1]), 10_000)[0] == 1001


def test_int_weights_paper_range():
    # costs in (0, 1] after prescaling -> weights in [1, alpha]
    wl = make_small(1)
    g = oracle.build(wl.row_ptr, wl.col_idx, wl.val, scale_rows=1)
    alpha = 10_000
    wg = oracle.int_weights(g.w, alpha)
    assert wg.min() >= 1 and wg.max() <= alpha
    with pytest.raises(oracle.OracleError):
        oracle.int_weights(np.array([0.5]), 0)
    with pytest.raises(oracle.OracleError):
        oracle.int_weights(np.array([-0.5]), 10)


@pytest.mark.parametrize("threads", [2, 3, 8])
def test_parallel_oracle_identical(threads):
    """orc_build_par (OpenMP row chunks) returns
    orc_build's outputs bit for bit, for any thread count and row range."""
    rng = np.random.default_rng(77 + threads)
    for cfg in (1, 4, 5):
        w = make_small(cfg)
        a, b = (0, w.n) if cfg != 5 else (123, w.n - 77)
        g1 = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol,
                          row_begin=a, row_end=b)
        gp = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol,
                          row_begin=a, row_end=b, threads=threads)
        assert np.array_equal(g1.row_ptr, gp.row_ptr) and np.array_equal(g1.col, gp.col)
        assert g1.w.tobytes() == gp.w.tobytes() and g1.diag.tobytes() == gp.diag.tobytes()
        assert np.array_equal(g1.nnzc, gp.nnzc)
    assert rng is not None


def test_full_size_golden_record():
    """tests/golden/full_size_digests.json (tools/make_full_golden.py, oracle
    only) covers configs 1-5; its totals agree with the closed forms of the
    stencil configs and its blocks tile the rows."""
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "full_size_digests.json")) as fh:
        gold = json.load(fh)
    assert all(str(c) in gold for c in (1, 2, 3, 4, 5))
    assert gold["2"]["graph_nnz"] == 11_980_004 and gold["3"]["graph_nnz"] == 190_322_400
    for c in (1, 2, 3, 4, 5):
        g = gold[str(c)]
        rows = [b["rows"] for b in g["blocks"]]
        assert rows[0][0] == 0 and rows[-1][1] == g["n"]
        assert all(r[1] == s[0] for r, s in zip(rows, rows[1:]))
        assert sum(b["nnz"] for b in g["blocks"]) == g["graph_nnz"]
        assert 0.0 <= g["cut"] <= g["total_weight"]
    # config 2 at full size through the oracle here: the recorded digests and cut
    w = make(2)
    a_hat = oracle.scale(w.row_ptr, w.val)[0]
    csc = oracle.transpose(w.n, w.n, w.row_ptr, w.col_idx, a_hat)
    import hashlib

    blk = gold["2"]["blocks"][5]
    a, b = blk["rows"]
    rp, col, wv, diag, _ = oracle.build_from_scaled(w.n, w.n, w.row_ptr, w.col_idx, a_hat, csc, w.drop_tol, a, b)
    h = hashlib.sha256()
    for x, dt in ((rp, "<i8"), (col, "<i4"), (wv, "<f8"), (diag, "<f8")):
        h.update(np.ascontiguousarray(x, dtype=dt).tobytes())
    assert h.hexdigest() == blk["sha256"]
