"""Summarise an ncu --set full report (raw page CSV) into the metrics this kernel is judged on.
Usage: ncu -i rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv"""
import csv
import sys

WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active",
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
        print(f"## {d.get('Kernel Name', '?')[:100]}")
        for k in WANT:
            if k in d:
                print(f"{k:70s} {d[k]:>22s} {u[k]}")
        st = []
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k].replace(",", ""))))
                except ValueError:
                    pass
        tot = sum(v for _, v in st) or 1.0
        print("stall samples (share):", ", ".join(f"{k} {v / tot:.1%}" for k, v in sorted(st, key=lambda t: -t[1])[:9]))


if __name__ == "__main__":
    main(sys.argv[1])
