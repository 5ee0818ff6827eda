"""Per CUDA source line: instructions executed and stall samples of one
kernel in an ncu report (needs -lineinfo and --import-source)."""
import csv
import io
import subprocess
import sys


def main(rep, kregex, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "--kernel-name",
                          f"regex:{kregex}", "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, recs, hdr = "", [], None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0] and r[0].isdigit():
            ie = hdr.index("Instructions Executed")
            sm = hdr.index("Warp Stall Sampling (All Samples)")
            try:
                recs.append((int(r[ie] or 0), int(r[sm] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
            except ValueError:
                pass
    ti = sum(x[0] for x in recs) or 1
    ts = sum(x[1] for x in recs) or 1
    print(f"total inst {ti} samples {ts}")
    for x in sorted(recs, key=lambda x: -x[0])[:int(top)]:
        print(f"{100 * x[0] / ti:5.1f}% inst {100 * x[1] / ts:5.1f}% stall  {x[2]:22s} {x[3]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
