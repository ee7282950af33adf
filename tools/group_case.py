"""One config-2 (sigma, m) group of 100 patterns through the group search, a few times (for ncu).
usage: python tools/group_case.py sigma m [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

s, m = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = torch.device("cuda:0")
n = 256 * synth.MiB
t = synth.text_torch(synth.raw_sigma_spec(s, (2, s)), 0, n, device=dev)
pats, _ = synth.extract_patterns_torch(t, (2, s, m), m, 100)
g = epsm.group(pats)
vals = g.index_values()
ix = epsm.eq_index(t, vals) if vals else None
occ = torch.zeros(100, dtype=torch.int64, device=dev)
g.count_async(t, occ, index=ix)
torch.cuda.synchronize()
cap = int(occ.max()) + 1
outs = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(100)]
for _ in range(reps):
    g.search_async(t, occ, outs=outs, index=ix)
torch.cuda.synchronize()
print("info", g.info(), "occ total", int(occ.sum()))
