"""Per-CTA timeline of back-to-back searches (run with EPSM_TRACE=16 in the environment)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sigma", type=int, default=256)
ap.add_argument("--m", type=int, default=32)
ap.add_argument("--n", type=int, default=256 * synth.MiB)
ap.add_argument("--count", action="store_true")
a = ap.parse_args()
assert os.environ.get("EPSM_TRACE"), "set EPSM_TRACE=16"
dev = torch.device("cuda:0")
t = synth.text_torch(synth.raw_sigma_spec(a.sigma, (2, a.sigma)), 0, a.n, device=dev)
R = 12
pats, _ = synth.extract_patterns_torch(t, (2, a.sigma, a.m), a.m, R)
plans = [epsm.plan(p) for p in pats]
out = torch.empty(a.n, dtype=torch.int64, device=dev)
occ = torch.zeros(R, dtype=torch.int64, device=dev)
for i, pl in enumerate(plans):     # warm-up (workspace allocation)
    (epsm.count_async(pl, t, occ[i:i + 1]) if a.count else epsm.search_async(pl, t, out, occ[i:i + 1]))
torch.cuda.synchronize()
L0 = epsm.launch_count()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i, pl in enumerate(plans):
    (epsm.count_async(pl, t, occ[i:i + 1]) if a.count else epsm.search_async(pl, t, out, occ[i:i + 1]))
e1.record()
torch.cuda.synchronize()
print(f"{'count' if a.count else 'search'} sigma={a.sigma} m={a.m} n={a.n >> 20} MiB: "
      f"{e0.elapsed_time(e1) * 1e3 / R:.1f} us per launch (events around {R} launches)")
tr = epsm.debug_trace()
slots = tr.shape[0]
names = ["start", "tma0", "tile0", "prod_end", "cons_end", "drain_end", "cta_end"]
prev_end = None
for k in range(R):
    L = (L0 + k) % slots
    d = tr[L].astype(np.int64)
    grid = int((d[:, 0] > 0).sum())
    d = d[:grid]
    t0 = d[:, 0].min()
    rel = (d[:, :7] - t0) / 1e3
    ends = d[:, 6].max()
    row = []
    for i, nm in enumerate(names):
        col = rel[:, i][d[:, i] > 0]
        if col.size:
            row.append(f"{nm} {np.percentile(col, 5):6.2f}/{np.median(col):6.2f}/{col.max():6.2f}")
    gap = f"gap_from_prev_end {(t0 - prev_end) / 1e3:6.2f}" if prev_end is not None else ""
    prev_end = ends
    span = (ends - t0) / 1e3
    print(f"launch {k:2d} grid {grid} span {span:6.2f} us {gap} chunks/cta {d[:, 7].min()}-{d[:, 7].max()}")
    print("    " + " | ".join(row))
