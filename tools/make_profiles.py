"""Copy one evidence run (tools/gpu_evidence.sh, gpurun_out/) into profiles/
under a round tag, and refresh profiles/ncu_summary.json (the per-launch DRAM
traffic bench.py reports as roofline.traffic) from the new ncu captures.

usage: python tools/make_profiles.py r02c
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")

# numeric kernel per config whose traffic bench.py reports (the dominant kernel
# of the path that config takes; config 4: the whole mixed pass's captured kernels)
NUMERIC = {2: ("full_c2", "k_num_pair<5>"), 3: ("full_c3", "k_num_pair<7>"), 5: ("full_c5", "k_row_win<0>")}
MIXED4 = ("full_c4", ("k_row_win<1>", "k_row_cta", "k_num_pair", "k_num_mid", "k_num_huge", "k_copy_rows"))


def summarise(rep):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                         capture_output=True, text=True).stdout
    return [json.loads(l) for l in out.splitlines() if l.strip().startswith("{")]


def main(tag):
    os.makedirs(P, exist_ok=True)
    copies = {"gputests.log": f"{tag}_gpu_tests.txt", "smoke.log": f"{tag}_smoke.txt",
              "bench_default.json": f"{tag}_bench_default.json", "bench_reference.json": f"{tag}_bench_reference.json",
              "rc_bench_all_configs.jsonl": f"{tag}_bench_all_configs.jsonl",
              "bench_2ranks_shared.json": f"{tag}_bench_2ranks_shared_gpu.json"}
    for src, dst in copies.items():
        if os.path.exists(os.path.join(G, src)):
            shutil.copy(os.path.join(G, src), os.path.join(P, dst))
    for c in (2, 3, 4, 5, 6, 7):
        csvp = os.path.join(G, f"launches_c{c}.csv")
        if os.path.exists(csvp):
            shutil.copy(csvp, os.path.join(P, f"{tag}_launches_config{c}.csv"))
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), csvp,
                            os.path.join(P, f"{tag}_launches_config{c}.md")], capture_output=True)
    summ = {}
    for name in ("full_c2", "full_c3", "full_c4", "full_c5", "full_c5t"):
        rep = os.path.join(G, name + ".ncu-rep")
        if os.path.exists(rep):
            rows = summarise(rep)
            summ[name] = rows
            cfg = name[len("full_c"):]
            with open(os.path.join(P, f"{tag}_ncu_full_config{cfg}.jsonl"), "w") as fh:
                for r in rows:
                    fh.write(json.dumps(r) + "\n")
    sp = os.path.join(P, "ncu_summary.json")
    d = json.load(open(sp)) if os.path.exists(sp) else {"numeric": {}}
    src = "profiles/{tag}_ncu_full_config{c}.jsonl (ncu --set full --clock-control none, bench.py --steps 2 --warmup 3 --config {c})"
    for c, (name, kern) in NUMERIC.items():
        rows = [r for r in summ.get(name, []) if kern in r["kernel"]]
        if rows:
            r = rows[0]
            d["numeric"][f"config{c}"] = {"dram_bytes": r["dram_rd"] + r["dram_wr"], "duration_us_cold": r["dur_us"],
                                          "kernel": "void " + kern if not r["kernel"].startswith("void") else r["kernel"],
                                          "source": src.format(tag=tag, c=c)}
    name, kerns = MIXED4
    rows = [r for r in summ.get(name, []) if any(k in r["kernel"] for k in kerns)]
    if rows:
        d["numeric"]["config4"] = {"dram_bytes": sum(r["dram_rd"] + r["dram_wr"] for r in rows),
                                   "duration_us_cold": round(sum(r["dur_us"] for r in rows), 3),
                                   "kernel": "mixed pass: " + " + ".join(sorted({r["kernel"].replace("void ", "") for r in rows})),
                                   "source": src.format(tag=tag, c=4)}
    json.dump(d, open(sp, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "rXX")
