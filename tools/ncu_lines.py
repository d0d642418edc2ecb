"""Map ncu per-SASS warp-stall samples onto CUDA source lines.

    ncu -i REP --page source --csv --print-source sass > sass.csv
    cuobjdump -xelf all paper_2208_14228_b200/_build/bt_mlp.cu.o; nvdisasm -g -fun KERNEL X.cubin > k.sass
    python tools/ncu_lines.py sass.csv k.sass paper_2208_14228_b200/csrc/bt_mlp.cu
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ia, iall, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lm, cur = {}, None
for line in open(sys.argv[2]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m:
        lm[int(m.group(1), 16)] = cur
base = int(data[0][ia], 16)
tot, byline = 0.0, collections.Counter()
for r in data:
    s = float(r[iall] or 0)
    tot += s
    byline[lm.get(int(r[ia], 16) - base)] += s
src = {sys.argv[3].split("/")[-1]: open(sys.argv[3]).read().split("\n")}
print("total samples", tot)
for k, v in byline.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 50):
    txt = src[k[0]][k[1] - 1].strip()[:90] if k and k[0] in src else ""
    print(f"{v:7.0f} {100 * v / tot:5.1f}% {str(k):28s} {txt}")
