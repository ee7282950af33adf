"""Run one (sigma, m) search of the bench workload a few times (for ncu / quick timing)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sigma", type=int, default=256)
ap.add_argument("--m", type=int, default=8)
ap.add_argument("--n", type=int, default=256 * synth.MiB)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--count", action="store_true")
ap.add_argument("--batch", type=int, default=0, help="searches per batch launch (0: single launches)")
ap.add_argument("--index", action="store_true", help="batch over an equality-mask index of the text")
a = ap.parse_args()
dev = torch.device("cuda:0")
t = synth.text_torch(synth.raw_sigma_spec(a.sigma, (2, a.sigma)), 0, a.n, device=dev)
pats, _ = synth.extract_patterns_torch(t, (2, a.sigma, a.m), a.m, a.reps)
out = torch.empty(a.n, dtype=torch.int64, device=dev)
occ = torch.zeros(1, dtype=torch.int64, device=dev)
plans = [epsm.plan(p) for p in pats]
for pl in plans:   # warm-up: workspace allocation happens on a plan's first call
    if a.count:
        epsm.count_async(pl, t, occ)
    else:
        epsm.search_async(pl, t, out, occ)
torch.cuda.synchronize()
if a.batch:
    # warm-up batch, then timed batches of a.batch searches each (one launch per batch)
    occb = torch.zeros(a.batch, dtype=torch.int64, device=dev)
    outs = [torch.empty(a.n // 2, dtype=torch.int64, device=dev) for _ in range(2)]
    ix = epsm.eq_index(t, epsm.index_values(plans)) if a.index else None
    groups = [plans[i:i + a.batch] for i in range(0, len(plans) - a.batch + 1, a.batch)]
    epsm.search_batch_async(groups[0], t, occb, outs=[outs[i % 2] for i in range(a.batch)], index=ix)
    torch.cuda.synchronize()
    for g in groups:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        epsm.search_batch_async(g, t, occb, outs=[outs[i % 2] for i in range(a.batch)], index=ix)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.batch
        print(f"sigma={a.sigma} m={a.m} batch of {a.batch}: {us:.1f} us per search  {a.n / us / 1e3:.1f} GB/s text")
    print("occ", occb.cpu().tolist()[:4])
    sys.exit(0)
evs = []
for pl in plans:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if a.count:
        epsm.count_async(pl, t, occ)
    else:
        epsm.search_async(pl, t, out, occ)
    e1.record()
    evs.append((e0, e1))
torch.cuda.synchronize()
for (e0, e1) in evs:
    us = e0.elapsed_time(e1) * 1e3
    print(f"sigma={a.sigma} m={a.m} {'count' if a.count else 'search'} {us:.1f} us  {a.n / us / 1e3:.1f} GB/s text")
print("occ", int(occ.item()))
