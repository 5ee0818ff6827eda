"""Per CUDA source line: instructions executed (per unit) and stall samples,
from an ncu report captured with --import-source (cuda,sass view)."""
import csv, io, subprocess, sys

rep, units = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
kre = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kre and kre.startswith("skip="):  # select the report's n-th launch instead of a name
    cmd += ["--launch-skip", kre[5:], "--launch-count", "1"]
elif kre:
    cmd += ["--kernel-name", f"regex:{kre}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
fname = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 10 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            ie = float(r[7] or 0); smp = float(r[4] or 0)
        except ValueError:
            continue
        res.append((ie, smp, fname, r[0], r[1].strip()[:90]))
ti = sum(x[0] for x in res); ts = sum(x[1] for x in res)
print(f"total inst {ti:.4g} ({ti/units:.1f}/unit), samples {ts:.0f}")
for ie, smp, f, ln, src in sorted(res, reverse=True)[:int(sys.argv[4]) if len(sys.argv) > 4 else 45]:
    print(f"{ie/units:8.1f} {100*smp/ts:5.1f}%  {f}:{ln}  {src}")
