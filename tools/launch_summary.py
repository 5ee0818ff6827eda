"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) into
per-kernel totals and shares of the step (cold-cache, serialised times)."""
import collections
import csv
import sys


def main(path, out_md=None):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    mine = {k: v for k, v in agg.items() if "rig::" in k}
    tot = sum(v[1] for v in mine.values())
    lines = ["| kernel | launches | total us | avg us | share of librig time |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(mine.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.1f} | {t / c:.2f} | {t / tot:.3f} |")
    other = {k: v for k, v in agg.items() if "rig::" not in k}
    for k, (c, t) in other.items():
        lines.append(f"| (not librig) `{k[:60]}` | {c} | {t:.1f} | {t / c:.2f} | - |")
    txt = "\n".join(lines)
    print(txt)
    if out_md:
        open(out_md, "w").write(txt + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
