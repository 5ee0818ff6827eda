"""Write tests/golden/full_size_digests.json: the ORACLE's G_RIP of every
BASELINE.json config at full size, as sha256 digests of fixed row blocks,
plus its cutsize.  Calls only oracle/ (and the seeded input generators); the
GPU path is never involved.  tests/test_gpu_fullsize.py compares the CUDA
path's graph block by block against these digests (bit-exact structure and
weights) and its cut within 1e-12.

    python tools/make_full_golden.py [--configs 1 2 3 4 5] [--threads N]

Block b covers rows [b*R, min(n, (b+1)*R)), R = ceil(n / BLOCKS).  Digest =
sha256(local row_ptr int64 || col int32 || w float64 || diag float64), all
little-endian.  Cut = math.fsum of the oracle's Neumaier cutsize of each
block (each block's own sum follows PAPER.md:393-405, eq. partcut).
"""
import argparse
import hashlib
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from rig_inputs import make  # noqa: E402

BLOCKS = 16
OUT = os.path.join(ROOT, "tests", "golden", "full_size_digests.json")


def input_digest(w):
    h = hashlib.sha256()
    for a in (w.row_ptr, w.col_idx, w.val, w.part):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def block_digest(rp_local, col, wv, diag):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rp_local, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(col, dtype="<i4").tobytes())
    h.update(np.ascontiguousarray(wv, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(diag, dtype="<f8").tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5])
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    args = ap.parse_args()
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    data["_about"] = ("oracle G_RIP of each BASELINE.json config at full size (rig_inputs.make): sha256 of "
                      "row blocks (local row_ptr i64 | col i32 | w f64 | diag f64), and the cutsize; written by "
                      "tools/make_full_golden.py, which calls only oracle/")
    for cfg in args.configs:
        t0 = time.time()
        w = make(cfg)
        n = w.n
        a_hat = oracle.scale(w.row_ptr, w.val)[0] if w.scale_rows else w.val
        csc = oracle.transpose(n, w.ncols, w.row_ptr, w.col_idx, a_hat)
        R = -(-n // BLOCKS)
        blocks, cuts, totals, nnz = [], [], [], 0
        for a in range(0, n, R):
            b = min(n, a + R)
            rp, col, wv, diag, _ = oracle.build_from_scaled(n, w.ncols, w.row_ptr, w.col_idx, a_hat, csc,
                                                            w.drop_tol, a, b, threads=args.threads)
            blocks.append({"rows": [a, b], "nnz": int(rp[-1]), "sha256": block_digest(rp, col, wv, diag)})
            c, tot, _intra = oracle.cutsize(rp, col, wv, w.part, w.K, row_begin=a)
            cuts.append(c)
            totals.append(tot)
            nnz += int(rp[-1])
        data[str(cfg)] = {"workload": w.recipe, "n": n, "input_sha256": input_digest(w), "rows_per_block": R,
                          "graph_nnz": nnz, "cut": math.fsum(cuts), "total_weight": math.fsum(totals),
                          "blocks": blocks}
        print(f"config {cfg}: n={n} graph nnz={nnz} cut={math.fsum(cuts):.17g} ({time.time() - t0:.1f}s)",
              flush=True)
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1)


if __name__ == "__main__":
    main()
