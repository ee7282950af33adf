"""Config-2 sweep, per (sigma, m): the group search (one pass per group of 100 patterns) against
the batch API (one pass per search, equality-mask index where it qualifies).  Diagnostics only.

usage: python tools/group_sweep.py [sigmas] [ms] [patterns]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

sigmas = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8,16,32,64,128,256").split(",")]
ms = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8,16,32").split(",")]
P = int(sys.argv[3]) if len(sys.argv) > 3 else 100
dev = torch.device("cuda:0")
n = 256 * synth.MiB
st = torch.cuda.current_stream()


def ev():
    return torch.cuda.Event(enable_timing=True)


print("sigma m  distinct(dense)  group_us  batch_us  occ_total  pos_GB  group_TBps_text")
tot_g = tot_b = 0.0
for s in sigmas:
    t = synth.text_torch(synth.raw_sigma_spec(s, (2, s)), 0, n, device=dev)
    for m in ms:
        pats, _ = synth.extract_patterns_torch(t, (2, s, m), m, P)
        g = epsm.group(pats)
        plans = [epsm.plan(p) for p in pats]
        occ = torch.zeros(P, dtype=torch.int64, device=dev)
        g.count_async(t, occ)
        torch.cuda.synchronize()
        cap = int(occ.max()) + 1
        outs = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(P)]
        occ_b = torch.zeros(P, dtype=torch.int64, device=dev)
        vals = epsm.index_values(plans)
        ix = epsm.eq_index(t, vals) if vals else None
        for _ in range(2):
            g.search_async(t, occ, outs=outs, index=ix)
            epsm.search_batch_async(plans, t, occ_b, outs=outs, index=ix)
        torch.cuda.synchronize()
        assert torch.equal(occ, occ_b), (s, m)
        e = [ev() for _ in range(4)]
        e[0].record(st)
        for _ in range(3):
            g.search_async(t, occ, outs=outs, index=ix)
        e[1].record(st)
        e[2].record(st)
        for _ in range(3):
            epsm.search_batch_async(plans, t, occ_b, outs=outs, index=ix)
        e[3].record(st)
        torch.cuda.synchronize()
        gu = e[0].elapsed_time(e[1]) * 1e3 / 3
        bu = e[2].elapsed_time(e[3]) * 1e3 / 3
        tot_g += gu
        tot_b += bu
        o = int(occ.sum())
        inf = g.info()
        print("%5d %2d %5d(%3d) %9.1f %9.1f %10d %7.2f %9.1f" % (
            s, m, inf["distinct"], inf["dense"], gu, bu, o, 8 * o / 1e9, P * n / (gu * 1e-6) / 1e12), flush=True)
        if ix is not None:
            ix.close()
        g.close()
        for pl in plans:
            pl.close()
        del outs
print("total group %.1f us, batch %.1f us" % (tot_g, tot_b))
