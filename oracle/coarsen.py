"""Oracle for SURVEY.md §8(f) f4: the first stage of a multilevel partitioner
on G_RIP -- heavy-edge matching and one coarsening step.  TEST
INFRASTRUCTURE ONLY: imported by tests/ (never by the product path).

The paper hands G_RIP with integer edge weights wgt = ceil(alpha * cost) to
METIS and proposes a parallel partitioner for the second
stage; it does not spell out the coarsening, so the
algorithm below is this repository's reading (R23-R25), written out
plainly with Python loops (small graphs only):

R23 matching, in rounds r = 0 .. rounds-1: every unmatched vertex v picks its
    heaviest unmatched neighbour (largest weight, ties to the smallest index;
    none: no pick); v and u match iff v picks u and u picks v.  Vertices
    matched in a round are fixed for the later rounds; the rest stay
    singletons.
R24 coarse vertices: the leader of v is min(v, match(v)) (v itself when
    unmatched); coarse ids number the leaders in ascending order; the coarse
    vertex weight is the sum of its members' weights.
R25 coarse edges: every fine edge (v, j) contributes wgt(v, j) to the coarse
    pair (cmap(v), cmap(j)); pairs with cmap(v) = cmap(j) (the contracted
    edge) are dropped; coarse rows list their neighbours ascending.  Integer
    weights: the sums are exact, so the result is independent of order.
"""
from __future__ import annotations

import numpy as np


def hem_match(row_ptr, col, wgt, rounds=4):
    """R23.  Returns match int32[n] (partner, or -1)."""
    n = len(row_ptr) - 1
    match = [-1] * n
    for _ in range(rounds):
        cand = [-1] * n
        for v in range(n):
            if match[v] >= 0:
                continue
            best_w, best_u = None, -1
            for p in range(row_ptr[v], row_ptr[v + 1]):
                u = int(col[p])
                if u == v or match[u] >= 0:
                    continue
                w = int(wgt[p])
                if best_u < 0 or w > best_w or (w == best_w and u < best_u):
                    best_w, best_u = w, u
            cand[v] = best_u
        new = 0
        for v in range(n):
            u = cand[v]
            if u >= 0 and cand[u] == v:
                match[v] = u
                new += 1
        if new == 0:
            break
    return np.array(match, dtype=np.int32)


def coarsen(row_ptr, col, wgt, match, vwgt=None):
    """R24-R25.  Returns (cmap int32[n], nc, crow_ptr int64[nc+1],
    ccol int32[], cwgt int64[], cvwgt int64[nc])."""
    n = len(row_ptr) - 1
    vw = [1] * n if vwgt is None else [int(x) for x in vwgt]
    lead = [v if match[v] < 0 else min(v, int(match[v])) for v in range(n)]
    leaders = sorted(set(lead))
    cid = {v: c for c, v in enumerate(leaders)}
    cmap = [cid[lead[v]] for v in range(n)]
    nc = len(leaders)
    cvw = [0] * nc
    rows = [dict() for _ in range(nc)]
    for v in range(n):
        c = cmap[v]
        cvw[c] += vw[v]
        for p in range(row_ptr[v], row_ptr[v + 1]):
            d = cmap[int(col[p])]
            if d == c:
                continue
            rows[c][d] = rows[c].get(d, 0) + int(wgt[p])
    crow_ptr = [0]
    ccol, cw = [], []
    for c in range(nc):
        for d in sorted(rows[c]):
            ccol.append(d)
            cw.append(rows[c][d])
        crow_ptr.append(len(ccol))
    return (np.array(cmap, dtype=np.int32), nc, np.array(crow_ptr, dtype=np.int64),
            np.array(ccol, dtype=np.int32), np.array(cw, dtype=np.int64), np.array(cvw, dtype=np.int64))
