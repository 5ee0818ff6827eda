"""Run the gather-only probe (rig_gather_probe: the numeric pass's A_hat^T
gather loop alone) on a BASELINE config, for ncu to capture.  With --summarize
it turns ncu CSV logs into profiles/<tag>_l2_gather_config<c>.jsonl."""
import argparse
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["gpu__time_duration.sum", "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
           "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "dram__bytes_read.sum", "l1tex__t_sector_hit_rate.pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def run(cfg):
    import torch

    from paper_1710_07769_b200 import rig
    from rig_inputs import make

    w = make(cfg)
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    torch.cuda.synchronize()
    print("checksum", rig.rig_gather_probe(A, w.scale_rows))


def summarize(log, cfg, tag, out_dir):
    txt = open(log).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    h = rows[0]
    vals = {}
    for r in rows[1:]:
        if len(r) < len(h) or "k_gather_probe" not in r[h.index("Kernel Name")]:
            continue
        vals[r[h.index("Metric Name")]] = r[h.index("Metric Value")].replace(",", "")
    rec = {"config": cfg, "kernel": "k_gather_probe", "source": os.path.basename(log)}
    for m in METRICS:
        if m in vals:
            rec[m] = float(vals[m])
    rd, hit = rec.get("lts__t_sectors_srcunit_tex_op_read.sum"), rec.get("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum")
    if rd:
        rec["l2_read_hit_rate_gathers_pct"] = 100.0 * hit / rd
    path = os.path.join(out_dir, f"{tag}_l2_gather_config{cfg}.jsonl")
    with open(path, "w") as fh:
        fh.write(json.dumps(rec) + "\n")
    print(json.dumps(rec))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--summarize", default=None, help="ncu csv log to summarize")
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    a = ap.parse_args()
    if a.summarize:
        summarize(a.summarize, a.config, a.tag, a.out)
    else:
        run(a.config)
