"""Device timeline of the bench step via torch.profiler (CUPTI): per-kernel
device time and GPU busy vs wall time per step.  Diagnostic only.

    python tools/timeline.py [--config 2] [--steps 5]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1710_07769_b200 import rig  # noqa: E402
from rig_inputs import make  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    w = make(args.config)
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    part = torch.as_tensor(w.part, device="cuda")
    cut = torch.empty(1, dtype=torch.float64, device="cuda")

    def step():
        return rig.rig_build_cut(A, part, w.K, 0, w.n, w.scale_rows, w.drop_tol, out=cut)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    # host cost of one call while the GPU is otherwise idle
    t0 = time.perf_counter()
    for _ in range(args.steps):
        g, _ = step()
        del g
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.steps
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            g, _ = step()
            del g
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    agg = {}
    t_first, t_last = None, None
    for e in evs:
        k = e.name[:70]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        s = e.time_range.start
        t_first = s if t_first is None else min(t_first, s)
        t_last = e.time_range.end if t_last is None else max(t_last, e.time_range.end)
    busy = sum(v[1] for v in agg.values()) / args.steps
    print(f"wall per step (no profiler): {wall * 1e6:.1f} us; GPU busy per step: {busy:.1f} us; "
          f"span per step under profiler: {(t_last - t_first) / args.steps:.1f} us")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:70s} n/step={c / args.steps:5.1f} us/step={t / args.steps:8.1f}")
    # CPU side: time spent in CUDA runtime API calls
    cpu = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda"):
            a = cpu.setdefault(e.name, [0, 0.0])
            a[0] += 1
            a[1] += e.cpu_time_total
    print("CUDA runtime API (host):")
    for k, (c, t) in sorted(cpu.items(), key=lambda x: -x[1][1])[:15]:
        print(f"  {k:40s} n/step={c / args.steps:5.1f} us/step={t / args.steps:8.1f}")


if __name__ == "__main__":
    main()
