"""f4 measurement: heavy-edge matching (4 rounds) and one coarsening step of
G_RIP (METIS weights ceil(1e4 * cost)) for a bench config, with
CUDA events on the launching stream; one JSON line per config.

    python tools/bench_f4.py [config ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1710_07769_b200 import rig  # noqa: E402
from rig_inputs import make  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2], out


def main(cfgs):
    for c in cfgs:
        w = make(c)
        A = rig.CSR(w.row_ptr, w.col_idx, w.val)
        g = rig.rig_build(A, w.scale_rows, w.drop_tol, 0)
        wg = rig.rig_int_weights(g.w, 10_000)
        rp, ci = g.row_ptr, g.col_idx
        vw = torch.as_tensor(w.row_ptr[1:] - w.row_ptr[:-1], device="cuda")
        t_m, m = timed(lambda: rig.rig_hem_match(rp, ci, wg, rounds=4))
        t_c, out = timed(lambda: rig.rig_coarsen(rp, ci, wg, m, vwgt=vw))
        matched = int((m >= 0).sum().item())
        print(json.dumps({"stage": "f4 heavy-edge matching + coarsening", "config": c, "n": g.n, "graph_nnz": g.nnz,
                          "match_ms": round(t_m, 4), "coarsen_ms": round(t_c, 4),
                          "match_edges_per_s": g.nnz / (t_m * 1e-3), "coarsen_edges_per_s": g.nnz / (t_c * 1e-3),
                          "matched_fraction": matched / max(g.n, 1), "coarse_n": out["n"], "coarse_nnz": out["nnz"],
                          "note": "coarsen_ms includes its two host synchronisations (coarse size, coarse nnz)"}))


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [2, 3])
