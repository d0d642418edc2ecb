"""Top warp-stall SASS instructions of an ncu report (with the instructions around each hotspot).

    python tools/ncu_sass_top.py REP [N] [CONTEXT]
"""
import csv
import subprocess
import sys

rep, N = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True, errors="replace").stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
h, d = rows[hi], rows[hi + 1:]
ia, isrc = h.index("Address"), h.index("Source")
iall, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(r[iall] or 0) for r in d) or 1.0
order = sorted(range(len(d)), key=lambda i: -float(d[i][iall] or 0))[:N]
print(f"total samples {tot:.0f}")
for i in order:
    if ctx:
        print("----")
        for r in d[max(0, i - ctx):i + 2]:
            print(f"   {r[ia][-5:]} {r[ie]:>9s} {r[iall]:>6s} {r[isrc][:100]}")
    else:
        r = d[i]
        print(f"{float(r[iall]) / tot * 100:5.1f}% {r[ia][-5:]} {r[ie]:>9s} {r[isrc][:100]}")
