"""Text kernels vs the equality-mask index, per (sigma, m) of BASELINE.json's config 2.

For each sigma: the 256 MiB text, `--patterns` extracted patterns per m, the index built once
over the values those patterns need (timed), then per m one batched search of all patterns
with and without the index (best of --reps).  Prints microseconds per search for both and
the index build time.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sigmas", default="2,4,8,16,32")
ap.add_argument("--ms", default="2,4,8,16,32")
ap.add_argument("--patterns", type=int, default=40)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda:0")
n = 256 * synth.MiB


def timed(fn, reps):
    best = None
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e3
        best = t if best is None or t < best else best
    return best


for s in [int(x) for x in a.sigmas.split(",")]:
    t = synth.text_torch(synth.raw_sigma_spec(s, (2, s)), 0, n, device=dev)
    groups = {}
    for m in [int(x) for x in a.ms.split(",")]:
        pats, _ = synth.extract_patterns_torch(t, (2, s, m), m, a.patterns)
        groups[m] = [epsm.plan(p) for p in pats]
    allp = [p for g in groups.values() for p in g]
    vals = epsm.index_values(allp)
    ix = epsm.EqIndex()
    build_us = timed(lambda: ix.build_async(t, vals), a.reps) if vals else 0.0
    print(f"sigma={s}: index of {len(vals)} values built in {build_us:.1f} us", flush=True)
    for m, plans in groups.items():
        occ = torch.zeros(len(plans), dtype=torch.int64, device=dev)
        epsm.search_batch_async(plans, t, occ)
        torch.cuda.synchronize()
        cap = int(occ.max().item()) + 1
        nbuf = min(len(plans), 80)
        pool = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(nbuf)]
        outs = [pool[j % nbuf] for j in range(len(plans))]
        occ_ref = occ.clone()
        t_text = timed(lambda: epsm.search_batch_async(plans, t, occ, outs=outs), a.reps) / len(plans)
        line = f"  m={m:2d}: text {t_text:8.2f} us/search"
        if vals:
            t_idx = timed(lambda: epsm.search_batch_async(plans, t, occ, outs=outs, index=ix), a.reps) / len(plans)
            same = torch.equal(occ, occ_ref)
            d = max(len(set(p.pattern)) for p in plans)
            line += f"   index {t_idx:8.2f} us/search   (max d={d}, occ equal: {same})"
        print(line, flush=True)
        del pool, outs
    ix.close()
    for p in allp:
        p.close()
    del t
    torch.cuda.empty_cache()
