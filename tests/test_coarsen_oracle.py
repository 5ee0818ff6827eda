"""Pins of the f4 oracle (oracle/coarsen.py, R23-R25) against
values fixed outside it: hand-worked small graphs, the dense integer product
W_c = P^T W P (off-diagonal), weight conservation, matching validity and the
fixpoint of the matching rule."""
import numpy as np
import pytest

from oracle.coarsen import coarsen, hem_match
from rig_inputs import from_triplets


def sym_graph(n, edges):
    """Symmetric CSR (int64 weights) from undirected (u, v, w) edges."""
    r, c, w = [], [], []
    for u, v, x in edges:
        r += [u, v]
        c += [v, u]
        w += [x, x]
    rp, ci, vv = from_triplets(n, n, np.array(r), np.array(c), np.array(w, dtype=np.float64))
    return rp, ci, vv.astype(np.int64)


def test_path_graph():
    rp, ci, w = sym_graph(4, [(0, 1, 5), (1, 2, 1), (2, 3, 5)])
    m = hem_match(rp, ci, w)
    assert list(m) == [1, 0, 3, 2]
    cmap, nc, crp, cci, cw, cvw = coarsen(rp, ci, w, m)
    assert list(cmap) == [0, 0, 1, 1] and nc == 2
    assert list(crp) == [0, 1, 2] and list(cci) == [1, 0] and list(cw) == [1, 1]
    assert list(cvw) == [2, 2]


def test_star_ties_to_smallest_index():
    # centre 0; leaves 1..4 with weights 3, 7, 7, 2: the centre takes leaf 2
    # (weight 7, the smaller index of the tie); leaves 1, 3, 4 stay single
    rp, ci, w = sym_graph(5, [(0, 1, 3), (0, 2, 7), (0, 3, 7), (0, 4, 2)])
    m = hem_match(rp, ci, w)
    assert list(m) == [2, -1, 0, -1, -1]
    cmap, nc, crp, cci, cw, cvw = coarsen(rp, ci, w, m, vwgt=[1, 2, 3, 4, 5])
    assert list(cmap) == [0, 1, 0, 2, 3] and nc == 4
    assert list(cci[crp[0]:crp[1]]) == [1, 2, 3] and list(cw[crp[0]:crp[1]]) == [3, 7, 2]
    assert list(cvw) == [1 + 3, 2, 4, 5]


def test_later_rounds_match_what_remains():
    # 0-1 (9) wins round 0; 2 picks 1 (weight 8) in round 0 but 1 is taken;
    # in round 1 vertex 2 picks 3 (weight 1) and 3 picks 2: matched
    rp, ci, w = sym_graph(4, [(0, 1, 9), (1, 2, 8), (2, 3, 1)])
    assert list(hem_match(rp, ci, w, rounds=1)) == [1, 0, -1, -1]
    assert list(hem_match(rp, ci, w, rounds=2)) == [1, 0, 3, 2]


@pytest.mark.parametrize("seed", range(6))
def test_random_graphs_against_dense_product(seed):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(5, 60))
    m_edges = int(rng.integers(n, 4 * n))
    edges = {}
    for _ in range(m_edges):
        u, v = map(int, rng.integers(0, n, 2))
        if u != v:
            edges[(min(u, v), max(u, v))] = int(rng.integers(1, 6))  # small range: many ties
    rp, ci, w = sym_graph(n, [(u, v, x) for (u, v), x in edges.items()])
    vw = rng.integers(1, 10, n)
    m = hem_match(rp, ci, w, rounds=64)
    # a valid matching of edges
    for v in range(n):
        if m[v] >= 0:
            assert m[m[v]] == v and m[v] != v
            assert m[v] in ci[rp[v]:rp[v + 1]]
    # fixpoint: one more round matches nothing new
    W = np.zeros((n, n), dtype=np.int64)
    for v in range(n):
        W[v, ci[rp[v]:rp[v + 1]]] = w[rp[v]:rp[v + 1]]
    cand = np.full(n, -1)
    for v in range(n):
        if m[v] < 0:
            nb = [(W[v, u], -u) for u in range(n) if W[v, u] > 0 and m[u] < 0]
            if nb:
                cand[v] = -max(nb)[1]
    assert not any(cand[v] >= 0 and cand[cand[v]] == v for v in range(n))
    # coarse graph = off-diagonal of P^T W P, exact integers
    cmap, nc, crp, cci, cw, cvw = coarsen(rp, ci, w, m, vwgt=vw)
    P = np.zeros((n, nc), dtype=np.int64)
    P[np.arange(n), cmap] = 1
    Wc = P.T @ W @ P
    np.fill_diagonal(Wc, 0)
    D = np.zeros((nc, nc), dtype=np.int64)
    for c in range(nc):
        D[c, cci[crp[c]:crp[c + 1]]] = cw[crp[c]:crp[c + 1]]
        assert np.all(np.diff(cci[crp[c]:crp[c + 1]]) > 0)
    np.testing.assert_array_equal(D, Wc)
    assert cvw.sum() == vw.sum()
    np.testing.assert_array_equal(cvw, P.T @ vw)
    # the contracted edges are exactly the matched pairs' weights
    inner = sum(W[v, m[v]] for v in range(n) if m[v] >= 0)
    assert W.sum() - inner == Wc.sum()
    # coarse ids ascend with the leaders
    lead = np.where(m < 0, np.arange(n), np.minimum(np.arange(n), m))
    assert np.all(np.diff(cmap[np.unique(lead)]) == 1)
