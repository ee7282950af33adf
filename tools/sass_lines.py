"""Aggregate an ncu SASS source-page CSV by CUDA source line (via nvdisasm line info).

usage: sass_lines.py <src.csv> <cubin> <mangled kernel name> [top]
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict

csv_path, cubin, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line_of = {}
cur = None
inside = False
for ln in dis.splitlines():
    if ln.startswith(".text.") or ".section\t.text." in ln or ln.startswith("\t.section\t.text"):
        inside = fn in ln
        cur = None
        continue
    if not inside:
        continue
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
E = "Instructions Executed"
agg_s, agg_e = defaultdict(int), defaultdict(int)
for k, r in enumerate(rows[2:]):
    key = line_of.get(16 * k, "?")
    agg_s[key] += int(r[ix[S]] or 0)
    agg_e[key] += int(r[ix[E]] or 0)
ts, te = sum(agg_s.values()), sum(agg_e.values())
print(f"samples {ts} warp-inst {te}")
src = {}
for key in sorted(agg_s, key=lambda k: -agg_s[k])[:top]:
    f, _, n = key.partition(":")
    print(f"{key:28s} {100 * agg_e[key] / te:5.1f}% inst {100 * agg_s[key] / ts:5.1f}% samples")
