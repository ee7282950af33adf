"""Separate host issue cost, per-launch fixed cost and steady-state rate of the search kernel."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
R = 100
for n in (256 * synth.MiB, 1024 * synth.MiB):
    t = synth.text_torch(synth.raw_sigma_spec(256, (2, 256)), 0, n, device=dev)
    pats, _ = synth.extract_patterns_torch(t, (2, 256, 8), 8, R)
    plans = [epsm.plan(p) for p in pats]
    out = torch.empty(1 << 20, dtype=torch.int64, device=dev)
    occ = torch.zeros(R, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream()
    for mode in ("search", "count"):
        def issue():
            for i, pl in enumerate(plans):
                if mode == "search":
                    epsm.search_async(pl, t, out, occ[i:i + 1], stream=s)
                else:
                    epsm.count_async(pl, t, occ[i:i + 1], stream=s)
        issue()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        issue()
        h1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        gpu_us = e0.elapsed_time(e1) * 1e3 / R
        host_us = (h1 - h0) * 1e6 / R
        # CUDA graph of the same R launches
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g, stream=torch.cuda.Stream()):
                s2 = torch.cuda.current_stream()
                for i, pl in enumerate(plans):
                    if mode == "search":
                        epsm.search_async(pl, t, out, occ[i:i + 1], stream=s2)
                    else:
                        epsm.count_async(pl, t, occ[i:i + 1], stream=s2)
            g.replay()
            torch.cuda.synchronize()
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            graph_us = e0.elapsed_time(e1) * 1e3 / R
        except Exception as ex:  # noqa: BLE001
            graph_us = f"graph failed: {ex}"
        print(f"n={n >> 20} MiB {mode}: stream {gpu_us:.1f} us/launch ({n / gpu_us / 1e3:.0f} GB/s), "
              f"host issue {host_us:.1f} us/call, graph {graph_us}")
