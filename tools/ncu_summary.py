"""Summarise an ncu report (``--set full``) into the numbers we judge kernels by.

usage: python tools/ncu_summary.py gpurun_out/x.ncu-rep [label] > profiles/x.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("Kernel Name", "kernel"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst issue %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_throttle / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "stall sleeping / issue"),
]


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    cols = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu summary: {label}\n")
    print(f"source: `{rep}` (ncu --set full --clock-control none)\n")
    print("| metric | " + " | ".join(f"launch {k}" for k in range(len(data))) + " |")
    print("|---|" + "---|" * len(data))
    for key, name in METRICS:
        if key not in cols:
            continue
        i = cols[key]
        unit = units[i] if i < len(units) else ""
        vals = [d[i] for d in data]
        if key == "Kernel Name":
            vals = [v[:40] for v in vals]
        print(f"| {name} ({unit}) | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
