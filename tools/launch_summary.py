"""Summarise an ncu launch list of bench.py (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv): per-launch lines of the repo's kernels, per-kernel shares, and
profiles/traffic.json (DRAM bytes per launch of the dominant kernel, read by bench.py).
usage: [LAST_N=n] python tools/launch_summary.py launches.csv out.txt [traffic.json]"""
import collections
import csv
import json
import sys

src, out_path = sys.argv[1], sys.argv[2]
tj = sys.argv[3] if len(sys.argv) > 3 else None
lines = [ln for ln in open(src) if ln.startswith('"')]
rows = collections.OrderedDict()
for r in csv.DictReader(lines):
    rows.setdefault((r["ID"], r["Kernel Name"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
# LAST_N=<n>: keep only the last n launches of the repo's kernels (the steps, not the setup's sizing pass)
import os
if os.environ.get("LAST_N"):
    keep = [k for k in rows if "epsm" in k[1] or "cg::" in k[1]][-int(os.environ["LAST_N"]):]
    rows = collections.OrderedDict((k, rows[k]) for k in keep)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0])   # launches, time, read, write, launches > 1 MB
with open(out_path, "w") as out:
    out.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
              "--clock-control none (cold-cache, serialised launches: shares, not absolutes)\n")
    out.write("# id kernel time_us dram_read_MB dram_write_MB\n")
    for (i, name), m in rows.items():
        if "epsm" not in name and "cg::" not in name:   # (the repo's kernels: namespace epsm, ncu
            continue                                    # shows epsm::cg as cg::)
        short = name.split("(")[0].replace("void ", "").replace("epsm::", "")
        t, rd, wr = m.get("gpu__time_duration.sum", 0), m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
        out.write(f"{i} {short[:70]} {t / 1e3:.1f} {rd / 1e6:.1f} {wr / 1e6:.1f}\n")
        a = agg[short.split("<")[0]]
        a[0] += 1
        a[1] += t
        a[2] += rd
        a[3] += wr
        a[4] += 1 if rd + wr > 1e6 else 0
    tot = sum(a[1] for a in agg.values())
    out.write("\n# per kernel (repo kernels only)\n")
    summ = {"source": out_path, "kernels": {}}
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.write(f"# {k}: launches {a[0]}, {a[1] / 1e6:.2f} ms ({100 * a[1] / tot:.1f}%), DRAM {a[2] / 1e9:.2f} GB "
                  f"read + {a[3] / 1e9:.2f} GB written, {(a[2] + a[3]) / a[0] / 1e6:.1f} MB per launch\n")
        summ["kernels"][k] = {"launches": a[0], "share": round(a[1] / tot, 4),
                              "dram_bytes_per_launch": int((a[2] + a[3]) / a[0]),
                              # (launches that moved > 1 MB: the step's launches, not the empty
                              # fan-outs of the bench's small warm-up / parity calls)
                              "dram_bytes_per_busy_launch": int((a[2] + a[3]) / max(a[4], 1)), "busy_launches": a[4]}
dom = max(summ["kernels"].items(), key=lambda x: x[1]["share"])
summ["dominant"] = dom[0]
summ["dram_bytes_per_launch"] = dom[1]["dram_bytes_per_busy_launch"]
summ["unit"] = ("DRAM bytes (read + write) per launch of the dominant kernel (" + dom[0] + "), ncu launch list of "
                "the bench, over its launches that moved > 1 MB")
if tj:
    json.dump(summ, open(tj, "w"), indent=1)
print(open(out_path).read().split("# per kernel")[1])
