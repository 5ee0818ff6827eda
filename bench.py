#!/usr/bin/env python
"""Benchmark: one step = the whole hot path over
one synthetic matrix resident in HBM: rig_build (scale, transpose, analyze,
symbolic, numeric fused with abs/drop/diag-strip, compaction if needed) +
rig_cutsize (+ NCCL allreduce of the cut when N > 1).

Workload (N=1, default): BASELINE.json configs[4] -- banded-plus-random,
n = 4,000,000 (the config with the most work: 2.19e9 products, 1.13e9 graph
entries).  --config selects another (1-7).  Metric: A.A^T
intermediate products per second (P / step time), plus build ms and the
numeric pass's fraction of the HBM roofline (measured copy bandwidth and the
8.0 TB/s spec).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]
N > 1: launch with torchrun (one rank per GPU); rows of C are sharded by
flop count (rig_row_split) and built by dist.build_cut_sharded (the cut is
allreduced over NCCL); the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "A·A^T intermediate products/s and row-graph build ms; % of HBM roofline"
L2_FLUSH_BYTES = 512 << 20
SPEC_HBM_GBS = 8000.0  # B200 HBM3e spec (north star: "~8 TB/s")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5, help="BASELINE.json config id (1-based); default configs[4]")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded oracle sample (cpu_baseline)")
    ap.add_argument("--ref-step-seconds", type=float, default=3.0, help="--impl reference: oracle work per step")
    ap.add_argument("--clock-ms", type=int, default=100, help="nvidia-smi sampling period (0: off)")
    ap.add_argument("--soak-seconds", type=float, default=1.5,
                    help="untimed steps before the timed region so clocks are sampled under load")
    return ap.parse_args()


def numeric_alg_bytes(n, nnz_a, nnz_c):
    """read A CSR + read A_hat^T CSC + read row_ptr_C +
    write C once = 24(n+1) + 24 nnzA + 12 nnzC (perfect L2 reuse of gathers)."""
    return 24 * (n + 1) + 24 * nnz_a + 12 * nnz_c


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload_label(w):
    if w.cfg_id <= 5:
        return f"{w.name} (BASELINE configs[{w.cfg_id - 1}])"
    return f"{w.name} (SURVEY 8(f) f3 stress config {w.cfg_id})"


def load_traffic(cfg):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the numeric
    kernel from the committed ncu --set full summary, if present."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        e = d.get("numeric", {}).get(f"config{cfg}")
        return (float(e["dram_bytes"]), e.get("source")) if e else (None, None)
    except Exception:
        return None, None


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index, period_ms=100):
        self.dev = dev_index
        self.period = max(int(period_ms), 20)
        self.proc = None
        self.lines = []
        self.mark = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", str(self.period),
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def begin_load(self):
        self.mark = time.time()

    def stop(self):
        end = time.time()
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, line in self.lines:
            if self.mark is None or t < self.mark or t > end + 0.2:
                continue
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class OracleSample:
    """The oracle as it stands (plain C, oracle/), on a bounded sample of the
    workload: rows [0, R) of G_RIP (dense-accumulator Gustavson + the cutsize
    of those rows), the scaling and CSC prepared once beforehand.  R is sized
    from a short calibration so one sample takes about `seconds`."""

    def __init__(self, w):
        import oracle

        self.o, self.w = oracle, w
        t0 = time.perf_counter()
        self.a_hat = oracle.scale(w.row_ptr, w.val)[0] if w.scale_rows else w.val
        self.csc = oracle.transpose(w.n, w.ncols, w.row_ptr, w.col_idx, self.a_hat)
        self.prep_s = time.perf_counter() - t0
        self.f = oracle.row_products(w.row_ptr, w.col_idx, self.csc[0])[0]
        self.fpre = np.concatenate([[0], np.cumsum(self.f)])

    def run(self, rows, threads):
        w = self.w
        t0 = time.perf_counter()
        rp, col, wv, _d, _n = self.o.build_from_scaled(w.n, w.ncols, w.row_ptr, w.col_idx, self.a_hat, self.csc,
                                                       w.drop_tol, 0, rows, threads=threads)
        self.o.cutsize(rp, col, wv, w.part, w.K)
        return time.perf_counter() - t0, int(self.fpre[rows])

    def rows_for(self, seconds, threads):
        n = self.w.n
        r = min(n, 2048)
        while True:
            t, P = self.run(r, threads)
            if r >= n or t >= 0.25 * seconds:
                break
            r = min(n, r * 4)
        rate = P / max(t, 1e-9)  # products/s
        want = rate * seconds
        return int(min(n, max(r, np.searchsorted(self.fpre, want, side="left"))))


def cpu_baseline(w, seconds):
    """cpu_baseline of the JSON line: the oracle on this host, 1 thread and all
    cores (os.sched_getaffinity), each on a bounded row sample (~seconds/2)."""
    import oracle

    S = OracleSample(w)
    allc = oracle.default_threads()
    out = {}
    for label, th in (("1thread", 1), ("all", allc)):
        R = S.rows_for(seconds / 2, th)
        t, P = S.run(R, th)
        out[label] = (P / t, R, t, P)
    v, R, t, P = out["all"]
    v1, R1, t1, P1 = out["1thread"]
    return {"value": v, "unit": "products/s", "cores": allc, "kind": "oracle",
            "sample": (f"rows [0, {R}) of {w.name} ({P} products, {t:.1f}s on {allc} threads; "
                       f"Gustavson + cutsize; scaling + CSC ({S.prep_s:.1f}s, 1 thread) prepared once)"),
            "value_1thread": v1, "sample_1thread": f"rows [0, {R1}) ({P1} products, {t1:.1f}s)",
            "cpu_model": cpu_model()}


def run_reference(args):
    """--impl reference: the CPU oracle (the only reference this tier has)
    timed as it stands on the host cores, on our arm's config / metric: each
    step builds a bounded row sample of the workload on all cores (sized to
    ~--ref-step-seconds)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from rig_inputs import make

    import oracle

    w = make(args.config)
    oracle.build_lib()
    S = OracleSample(w)
    th = oracle.default_threads()
    R = S.rows_for(args.ref_step_seconds, th)
    for _ in range(max(0, min(args.warmup, 1))):
        S.run(R, th)
    times, P = [], 0
    for _ in range(args.steps):
        t, P = S.run(R, th)
        times.append(t)
    t = sum(times) / len(times)
    v = P / t
    sample = (f"rows [0, {R}) of {w.name} per step ({P} products; Gustavson + cutsize on {th} threads; "
              f"scaling + CSC prepared once, {S.prep_s:.1f}s)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "products/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_label(w), "n": w.n, "nnz_A": w.nnz, "K": w.K,
                       "sample_rows": R, "sample_products": P},
            "cpu_baseline": {"value": v, "unit": "products/s", "cores": th, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": "products/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    # BENCH_SHARE_GPU=1 / BENCH_DIST_BACKEND=gloo: exercise the N > 1 code path
    # on a one-GPU box (every rank on cuda:0, gloo); the numbers mean nothing then
    if os.environ.get("BENCH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_1710_07769_b200 import dist as rdist
    from paper_1710_07769_b200 import rig
    from rig_inputs import make

    w = make(args.config)
    stream = torch.cuda.current_stream()
    A = rig.CSR(w.row_ptr, w.col_idx, w.val)
    part = torch.as_tensor(w.part, device="cuda")
    split = rig.rig_row_split(A, world) if world > 1 else [0, w.n]
    rb, re = split[rank], split[rank + 1]
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")

    cut_buf = torch.empty(1, dtype=torch.float64, device="cuda")

    def step():
        # the whole hot path through the C ABI: a1-a6 (build) + a7 (cutsize);
        # N > 1: this rank's shard, then a8 (NCCL allreduce of the partial cuts)
        if world > 1:
            g, cut, _ = rdist.build_cut_sharded(A, part, w.K, w.scale_rows, w.drop_tol, split=split)
            return g, cut
        return rig.rig_build_cut(A, part, w.K, rb, re, w.scale_rows, w.drop_tol, out=cut_buf)

    # warm-up
    for _ in range(max(args.warmup, 3)):
        g, cut = step()
    torch.cuda.synchronize()
    nnz_local = g.nnz
    # products of this shard / of the whole matrix (plan query == oracle-free count)
    plan = rig.Plan(A, w.scale_rows, w.drop_tol, 0, rb, re)
    P_local = plan.products
    plan.destroy()
    P_total = P_local
    g_total = nnz_local
    if world > 1:
        t = torch.tensor([P_local, nnz_local], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        P_total, g_total = int(t[0]), int(t[1])
    # structural nnz(C) incl. diagonal = graph nnz + nonempty rows when nothing was dropped
    nnz_c = g_total + int((np.diff(w.row_ptr) > 0).sum())

    clocks = ClockSampler(local, args.clock_ms)
    if args.clock_ms > 0:
        clocks.start()
    clocks.begin_load()
    t_end = time.time() + args.soak_seconds
    while time.time() < t_end:
        flush.zero_()
        step()
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps, L2 flushed between steps.  Only the
    # numeric pass and its dominant kernel carry CUDA events (on the stream
    # they are launched on); the Python cyclic GC is paused so harness pauses
    # do not land in a step.
    import ctypes
    import gc

    PASS_NUMERIC, PASS_KERNEL = 7, 11
    rig.lib.rig_profile_read(None, None)
    rig.lib.rig_profile_enable((1 << PASS_NUMERIC) | (1 << PASS_KERNEL))
    launches0 = rig.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    gc.collect()
    gc.disable()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        g, cut = step()
        ev[k][1].record(stream)
        del g
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    gc.enable()
    launches = rig.launch_count() - launches0
    rig.lib.rig_profile_enable(0)
    pms = (ctypes.c_double * 13)()
    pcnt = (ctypes.c_int64 * 13)()
    rig.lib.rig_profile_read(pms, pcnt)
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    my_ms = sum(step_ms) / len(step_ms)
    num_ms = pms[PASS_NUMERIC] / max(pcnt[PASS_NUMERIC], 1)
    ker_ms = pms[PASS_KERNEL] / max(pcnt[PASS_KERNEL], 1)
    # per-pass breakdown from separate (untimed) profiled steps
    rig.lib.rig_profile_enable(1)
    nprof = max(3, min(args.steps, 10))
    for _ in range(nprof):
        flush.zero_()
        g, _c = step()
        del g
    torch.cuda.synchronize()
    rig.lib.rig_profile_enable(0)
    rig.lib.rig_profile_read(pms, pcnt)
    pass_ms = {rig.lib.rig_pass_name(i).decode(): pms[i] / nprof for i in range(13) if pcnt[i]}
    if dist:
        t = torch.tensor([my_ms, num_ms, ker_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        my_ms, num_ms, ker_ms = float(t[0]), float(t[1]), float(t[2])
    cut_val = float(cut.item())

    # ---- device memory of one build (library pool high-water mark; the
    # inputs A and part live in torch's allocator, the rest in the pool)
    torch.cuda.synchronize()
    rig.rig_mem_stats(reset=True)
    g, _c = step()
    torch.cuda.synchronize()
    pool_now, pool_high = rig.rig_mem_stats()
    a_bytes = 8 * (w.n + 1) + 12 * w.nnz
    csc_bytes = 8 * (w.ncols + 1) + 12 * (w.nnz + w.ncols)
    graph_bytes = 8 * (re - rb + 1) + 12 * g.nnz
    del g
    mem = {"pool_high_gb": pool_high / 1e9, "inputs_gb": (a_bytes + 4 * w.n) / 1e9,
           "a_csc_graph_gb": (a_bytes + csc_bytes + graph_bytes) / 1e9,
           "ratio": (pool_high + a_bytes + 4 * w.n) / (a_bytes + csc_bytes + graph_bytes),
           "note": "peak = library pool high-water mark during one build (workspaces + graph) + inputs; "
                   "ratio against A + CSC of A_hat + the exact graph"}

    # ---- e2e through the C ABI from pinned host buffers (N=1 path)
    e2e = None
    if world == 1:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hrp, hci, hv, hpart = pin(w.row_ptr), pin(w.col_idx), pin(w.val), pin(w.part)
        orp = torch.empty(w.n + 1, dtype=torch.int64).pin_memory()
        ocol = torch.empty(max(g_total, 1), dtype=torch.int32).pin_memory()
        ow = torch.empty(max(g_total, 1), dtype=torch.float64).pin_memory()
        for _ in range(2):
            rig.rig_build_host(hrp, hci, hv, w.n, w.scale_rows, w.drop_tol, 0, hpart, w.K, orp, ocol, ow)
        e_ms = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            nn, ccut = rig.rig_build_host(hrp, hci, hv, w.n, w.scale_rows, w.drop_tol, 0, hpart, w.K, orp, ocol, ow)
            b.record(stream)
            torch.cuda.synchronize()
            e_ms.append(a.elapsed_time(b))
        em = sum(e_ms) / len(e_ms)
        h2d = 8 * (w.n + 1) + 12 * w.nnz + 4 * w.n
        d2h = 8 * (w.n + 1) + 12 * nn + 8
        e2e = {"value": P_total / (em * 1e-3), "unit": "products/s", "ms_per_step": em, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peak, peak_src = load_peaks()
    alg = numeric_alg_bytes(w.n, w.nnz, nnz_c) / max(world, 1) if world > 1 else numeric_alg_bytes(w.n, w.nnz, nnz_c)
    path = rig.last_path()
    roof_ms = ker_ms if path in ("merge", "rowwin") else num_ms
    roof_kernel = {
        "merge": "k_num_pair (a5+a6 fused merge path, two lanes per row, all rows; CUDA events around the launch)",
        "rowwin": "k_row_win (a5+a6(+a7 partials) for every row, look-back placement; CUDA events around the launch)",
    }.get(path, "numeric pass (k_num_mid + k_num_huge + k_num_pair + k_copy_rows; CUDA events around the pass)")
    achieved = alg / (roof_ms * 1e-3) / 1e9
    traffic, traffic_src = load_traffic(args.config)
    line = {
        "metric": METRIC,
        "value": P_total / (my_ms * 1e-3),
        "unit": "products/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": my_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_label(w), "n": w.n, "nnz_A": w.nnz,
                   "products": P_total, "nnz_C": nnz_c, "graph_nnz": g_total, "K": w.K,
                   "scale_rows": w.scale_rows, "drop_tol": w.drop_tol,
                   "l2": f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write)",
                   "parallelism": f"rows of C sharded over {world} GPU(s), flop-balanced; NCCL allreduce of cut"
                   if world > 1 else "1 GPU"},
        "build_ms": my_ms - pass_ms.get("cutsize", 0.0),
        "numeric_ms": num_ms,
        "numeric_kernel_ms": ker_ms,
        "step_ms_min": min(step_ms),
        "step_ms_max": max(step_ms),
        "step_ms_median": statistics.median(step_ms),
        "pass_ms": pass_ms,
        "cut": cut_val,
        "roofline": {"bound": "hbm", "kernel": roof_kernel, "duration_ms": roof_ms,
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_spec": SPEC_HBM_GBS, "frac_spec": achieved / SPEC_HBM_GBS,
                     "traffic": traffic, "alg_bytes": alg,
                     "alg_bytes_formula": ("SURVEY §8(d) F1 = 24(n+1) + 24 nnzA + 12 nnzC per launch "
                                           "(nnzC = graph nnz + nonempty rows; entries dropped by drop_tol not counted)"),
                     "peak_source": peak_src, "traffic_source": traffic_src},
        "numeric_path": path,
        "gpu_launches": launches,
        "clocks": clk,
        "device_memory": mem,
    }
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
