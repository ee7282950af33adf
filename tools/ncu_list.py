"""Condense an `ncu --csv --metrics ...` launch list: one line per launch of the repo's kernels
(name shortened), metrics side by side.  usage: python tools/ncu_list.py file.csv [filter]"""
import csv
import sys
from collections import OrderedDict

rows = OrderedDict()
flt = sys.argv[2] if len(sys.argv) > 2 else "epsm"
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    name = r.get("Kernel Name", "")
    if flt not in name:
        continue
    key = (r["ID"], name)
    rows.setdefault(key, {})[r["Metric Name"]] = r["Metric Value"]
for (i, name), mets in rows.items():
    short = name.split("(")[0].replace("void ", "").replace("epsm::", "")[:60]
    t = float(mets.get("gpu__time_duration.sum", "0").replace(",", ""))
    rd = float(mets.get("dram__bytes_read.sum", "0").replace(",", ""))
    wr = float(mets.get("dram__bytes_write.sum", "0").replace(",", ""))
    print(f"{i:>5} {short:60s} {t/1e3:10.1f} us  rd {rd/1e6:9.1f} MB  wr {wr/1e6:9.1f} MB")
