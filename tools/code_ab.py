"""Time the bench's group call for some (sigma, m) of config 2 (256 MiB texts, 100 extracted
patterns, the library's dense split over the equality-mask index), as bench.py runs it.
A/B of the code-mode kernels: run once with EPSM_CODE_CG=0 (general kernels) and once without.

usage: python tools/code_ab.py "2:8,4:4,16:2" [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

cases = [tuple(int(x) for x in c.split(":")) for c in sys.argv[1].split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda:0")
n = 256 * synth.MiB
texts = {}
for s, m in cases:
    if s not in texts:
        texts[s] = synth.text_torch(synth.raw_sigma_spec(s, (2, s)), 0, n, device=dev)
    t = texts[s]
    pats, _ = synth.extract_patterns_torch(t, (2, s, m), m, 100)
    g = epsm.group(pats)
    vals = g.index_values()
    ix = epsm.eq_index(t, vals) if vals else None
    occ = torch.zeros(100, dtype=torch.int64, device=dev)
    g.count_async(t, occ, index=ix)
    torch.cuda.synchronize()
    cap = int(occ.max()) + 1
    outs = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(100)]
    g.search_async(t, occ, outs=outs, index=ix)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.search_async(t, occ, outs=outs, index=ix)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    print(f"sigma={s:4d} m={m:3d} passes={g.info()['passes']} us={us:9.1f} occ={int(occ.sum())}", flush=True)
    g.close()
    if ix is not None:
        ix.close()
