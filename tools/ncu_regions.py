"""Per-source-line cycle attribution from an ncu warp-sampling SASS page.

    python tools/ncu_regions.py sass.csv kernel.sass src.cu [N]
cycles per warp-step = samples / (samples-per-issue * warp-steps), where the
warp-step count is the execution count of the first SYNCS.PHASECHK (once per
warp per step) and samples-per-issue = stall_selected / instructions executed.
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ia, isrc, iall = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
isel, iex = hdr.index("stall_selected"), hdr.index("Instructions Executed")
base = int(data[0][ia], 16)


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


lm, cur = {}, None
for line in open(sys.argv[2]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m:
        lm[int(m.group(1), 16)] = cur
k = sum(f(r[isel]) for r in data) / sum(f(r[iex]) for r in data)
steps_warps = f([r for r in data if "PHASECHK" in r[isrc]][0][iex])
norm = k * steps_warps
src_name = sys.argv[3].split("/")[-1]
src = open(sys.argv[3]).read().split("\n")
agg = collections.Counter()
for r in data:
    l = lm.get(int(r[ia], 16) - base)
    key = l[1] if l and l[0] == src_name else (("lib:" + l[0]) if l else "?")
    agg[key] += f(r[iall])
print(f"cycles per warp-step (all warps averaged): {sum(agg.values()) / norm:.0f}")
for key, v in sorted(agg.items(), key=lambda x: -x[1])[: int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    txt = src[key - 1].strip()[:88] if isinstance(key, int) else ""
    print(f"{v / norm:8.1f} {str(key):26s} {txt}")
