"""Summarise an `ncu --page source --csv --print-source sass` export: top instructions by
stall samples, with their dominant stall reasons (reads only the CSV)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
tot_s = sum(int(r[ix[S]] or 0) for r in data)
tot_i = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
print("samples", tot_s, "warp-inst", tot_i)
stalls = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
agg = {h: sum(int(r[ix[h]] or 0) for r in data) for h in stalls}
print("stall totals:", ", ".join(f"{h[6:]} {100*v/tot_s:.1f}%" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, r in enumerate(data):
    r.append(k)
top = sorted(data, key=lambda r: -int(r[ix[S]] or 0))[:n]
for r in top:
    s = int(r[ix[S]])
    det = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    print(f"{r[-1]:5d} {s:6d} {100*s/tot_s:5.1f}% ex={r[ix['Instructions Executed']]:>8}", r[1].strip()[:58], det)
