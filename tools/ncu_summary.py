"""Summarise an ncu --set full report (raw page) into the metrics we track."""
import csv
import io
import json
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ"),
    ("launch__registers_per_thread", "regs"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("smsp__inst_executed.sum", "inst"),
    ("launch__grid_size", "grid"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_rd_sect"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "l2_wr_sect"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_lsb"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
]


def scale(v, unit):
    f = float(v.replace(",", ""))
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    return f * mul.get(unit, 1)


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for d in rows[2:]:
        name = d[h.index("Kernel Name")]
        e = {"kernel": name.split("(")[0]}
        for m, k in WANT:
            if m in h:
                i = h.index(m)
                try:
                    e[k] = scale(d[i], u[i])
                except ValueError:
                    e[k] = d[i]
        res.append(e)
    for e in res:
        print(json.dumps(e))


if __name__ == "__main__":
    main(sys.argv[1])
