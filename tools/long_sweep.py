"""Long patterns (m > 32) on a 1 GiB genome-like text: us per search (10 patterns extracted from
the text, one launch each, CUDA events), text GB/s.  Diagnostics; run twice with and without
EPSM_LONG_STRIDE=0 for the A/B of EPSMc's sampling stride.  usage: python tools/long_sweep.py [ms]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

ms = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "33,48,64,128,256,1024,4096").split(",")]
n = 1 << 30
dev = torch.device("cuda:0")
t = synth.text_torch(synth.uniform_spec(synth.ACGT, (3, 0)), 0, n, device=dev)
pos = torch.empty(1 << 20, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream()
print(" m   L   us/search  text_GB/s  occ")
for m in ms:
    pats, _ = synth.extract_patterns_torch(t, (3, 0, m), m, 10)
    plans = [epsm.plan(p) for p in pats]
    occ = torch.zeros(len(plans), dtype=torch.int64, device=dev)
    for j, pl in enumerate(plans):
        epsm.search_async(pl, t, pos, occ[j:j + 1])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for j, pl in enumerate(plans):
        epsm.search_async(pl, t, pos, occ[j:j + 1])
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / len(plans)
    L = 16 * (m // 16 - 1) if m >= 64 else 0
    print("%4d %4d %10.1f %10.1f %s" % (m, L, us, n / (us * 1e-6) / 1e9, occ.tolist()[:3]), flush=True)
    for pl in plans:
        pl.close()
