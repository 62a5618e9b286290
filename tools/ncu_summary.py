"""Summarize `ncu --page raw --csv` exports into a compact markdown table.

    python tools/ncu_summary.py profiles/r1_*_raw.csv > profiles/r1_summary.md
"""

import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "regs/thread"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st conflicts"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "mio_throttle", "lg_throttle",
          "math_pipe_throttle", "not_selected", "selected", "no_instructions", "dispatch_stall"]


def main(paths):
    for path in paths:
        with open(path) as f:
            rows = list(csv.reader(f))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        print(f"### {path}\n")
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            print(f"**{name[:90]}** (grid {r[hdr.index('Grid Size')] if 'Grid Size' in hdr else '?'})\n")
            print("| metric | value |\n|---|---|")
            for k, label in KEYS:
                if k in hdr and r[hdr.index(k)] not in ("", "n/a"):
                    print(f"| {label} | {r[hdr.index(k)]} {units[hdr.index(k)]} |")
            tot = hdr.index("smsp__pcsamp_sample_count") if "smsp__pcsamp_sample_count" in hdr else None
            if tot is not None:
                n = float(r[tot].replace(",", "") or 1)
                parts = []
                for s in STALLS:
                    k = f"smsp__pcsamp_warps_issue_stalled_{s}"
                    if k in hdr and r[hdr.index(k)]:
                        parts.append((float(r[hdr.index(k)].replace(",", "")) / n, s))
                parts.sort(reverse=True)
                print("| top stall samples | " + ", ".join(f"{s} {100 * v:.0f}%" for v, s in parts[:4]) + " |")
            print()


if __name__ == "__main__":
    main(sys.argv[1:])
