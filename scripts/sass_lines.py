"""Per-source-line warp instruction counts of an ncu capture.

ncu's SASS source page (Instructions Executed per instruction) joined with the
line table of the same build (nvdisasm -g of the cubin): argv[1] the .ncu-rep,
argv[2] the nvdisasm -g listing, argv[3] the kernel's mangled name.
"""
import collections
import csv
import re
import subprocess
import sys

rep, listing, name = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
iE = hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
cnt = [int(r[iE]) for r in data]
stall = [int(r[iW]) for r in data]
lines = {}
cur = None
inside = False
for ln in open(listing):
    if ln.startswith(".text." + name + ":"):
        inside = True
        continue
    if inside and ln.startswith(".text.") and not ln.startswith(".text." + name):
        break
    if not inside:
        continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        lines[int(m.group(1), 16) // 16] = cur
agg = collections.Counter()
aggw = collections.Counter()
for i, c in enumerate(cnt):
    agg[lines.get(i)] += c
    aggw[lines.get(i)] += stall[i]
tot, totw = sum(cnt), sum(stall)
print(f"total {tot} warp instructions, {totw} stall samples, {len(cnt)} SASS / {len(lines)} mapped")
for k, v in agg.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 40):
    print(f"{str(k):48s} {v:11d} {100 * v / tot:5.1f}%  stall {100 * aggw[k] / totw:5.1f}%")
