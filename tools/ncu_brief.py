"""One-screen summary of an ncu report: duration, DRAM bytes and throughput, occupancy, top stalls.

    python tools/ncu_brief.py REP [REP ...]
"""
import csv
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "MB"), ("dram__bytes_write.sum", "MB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"), ("launch__registers_per_thread", ""),
        ("launch__grid_size", ""), ("launch__block_size", ""), ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
        ("smsp__inst_executed.sum", ""), ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", ""),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "%"),
        ("launch__shared_mem_per_block_dynamic", "")]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    un = dict(zip(h, u))
    print(f"== {rep}: {d.get('Kernel Name', '')[:100]}")
    for k, _ in KEYS:
        if k in d:
            print(f"  {k:66s} {d[k]:>14s} {un.get(k, '')}")
    st = sorted(((float(d[k].replace(',', '') or 0), k) for k in d
                 if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                reverse=True)[:6]
    print("  stalls: " + ", ".join(f"{k[34:-27]} {x:.2f}" for x, k in st))
