"""Summarise an ncu --set full report (raw page) into the metrics we track:
duration, DRAM bytes/throughput, cache hit rates, occupancy, issue rate and
the top stall reasons (warps stalled per issue)."""
import csv
import io
import json
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "dur_us"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ"),
    ("launch__occupancy_limit_registers", "occ_lim_reg"),
    ("launch__occupancy_limit_shared_mem", "occ_lim_smem"),
    ("launch__registers_per_thread", "regs"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("smsp__inst_executed.sum", "inst"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_rd_sect"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "l2_wr_sect"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "gld_req"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "gld_sect"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
]
STALL = "smsp__average_warps_issue_stalled_"


def scale(v, unit):
    f = float(v.replace(",", ""))
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
           "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return f * mul.get(unit, 1)


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for d in rows[2:]:
        name = d[h.index("Kernel Name")]
        e = {"kernel": name.split("(")[0]}
        for m, k in WANT:
            if m in h:
                i = h.index(m)
                try:
                    e[k] = round(scale(d[i], u[i]), 3)
                except ValueError:
                    e[k] = d[i]
        st = {}
        for i, m in enumerate(h):
            if m.startswith(STALL) and m.endswith("_per_issue_active.ratio"):
                try:
                    st[m[len(STALL):-len("_per_issue_active.ratio")]] = float(d[i])
                except ValueError:
                    pass
        e["stalls"] = {k: round(v, 2) for k, v in sorted(st.items(), key=lambda x: -x[1])[:5]}
        print(json.dumps(e))


if __name__ == "__main__":
    main(sys.argv[1])
