"""Key metrics and stall reasons of each kernel in an ncu report (raw page)."""
import csv
import io
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__occupancy_limit_shared_mem',
        'launch__occupancy_limit_registers', 'launch__registers_per_thread', 'launch__grid_size',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__t_sector_hit_rate.pct',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__t_sector_hit_rate.pct']


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for v in rows[2:]:
        print("==", v[h.index("Kernel Name")][:60])
        for w in WANT:
            if w in h:
                print(f"  {w:62s} {v[h.index(w)]}")
        st = [(float(v[i]), n) for i, n in enumerate(h) if n.startswith('smsp__average_warps_issue_stalled_')
              and n.endswith('_per_issue_active.ratio') and v[i] not in ('', 'n/a')]
        print("  stalls:", ", ".join(f"{n[34:-23]}={x:.2f}" for x, n in sorted(st, reverse=True)[:7]))


if __name__ == "__main__":
    main(sys.argv[1])
