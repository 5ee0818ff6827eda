"""Hot SASS regions of one kernel in an ncu report: instruction share and
stall-sample share per window of W instructions (needs --import-source)."""
import csv
import io
import subprocess
import sys


def main(rep, kregex, skip=0, W=24, thresh=0.03):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kregex}",
                          "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if "Instructions Executed" in r][0]
    h = rows[hi]
    ie, src, smp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0

    data = [(num(r[ie]), num(r[smp]), r[src].strip()) for r in rows[hi + 1:] if len(r) > ie]
    # the csv repeats the listing per source view; keep the first copy
    tot, tots = sum(d[0] for d in data), sum(d[1] for d in data)
    print(f"inst {tot} samples {tots} sass {len(data)}")
    for s0 in range(0, len(data), W):
        blk = data[s0:s0 + W]
        a, b = sum(d[0] for d in blk), sum(d[1] for d in blk)
        if a > tot * thresh or b > tots * thresh:
            print(s0, f"{100 * a / tot:5.1f}% inst {100 * b / tots:5.1f}% stall |", " | ".join(d[2][:30] for d in blk[::4]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
