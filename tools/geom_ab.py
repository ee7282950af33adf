"""A/B of a group's geometry (the cost model's choice vs the forced code mode) on config-2 texts.
usage: python tools/geom_ab.py sigma:m [sigma:m ...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
n = 256 * synth.MiB
st = torch.cuda.current_stream()
for arg in sys.argv[1:]:
    s, m = (int(x) for x in arg.split(":"))
    t = synth.text_torch(synth.raw_sigma_spec(s, (2, s)), 0, n, device=dev)
    pats, _ = synth.extract_patterns_torch(t, (2, s, m), m, 100)
    for mode in ("auto", "code"):
        g = epsm.group(pats).set_dense(0)
        if mode == "code":
            try:
                g.set_geometry(m, 0)
            except epsm.EpsmError:
                print(s, m, "code mode n/a")
                continue
        occ = torch.zeros(100, dtype=torch.int64, device=dev)
        g.count_async(t, occ)
        torch.cuda.synchronize()
        outs = [torch.empty(int(occ.max()) + 1, dtype=torch.int64, device=dev) for _ in range(100)]
        g.search_async(t, occ, outs=outs)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            g.search_async(t, occ, outs=outs)
        e1.record(st)
        torch.cuda.synchronize()
        print(s, m, mode, g.info()["passes"], round(e0.elapsed_time(e1) * 1e3 / 3, 1), "us", flush=True)
        g.close()
