"""Throughput of the batched search on BASELINE.json's other configs (3a, 3b, 4, 5a, 5b).

bench.py measures config 2 (the metric's sweep); this tool times, per (config, m), one call
of epsm_search_batch_async over the config's text with `--patterns` extracted patterns,
every search writing all its positions into its own buffer, and prints one JSON object:
per (config, m) microseconds per search, text GB/s, algorithmic GB/s (text + 8 B per
position) and the total occ.  Inputs are the seeded synthetic stand-ins of synth/.
Config 5a (8 GiB) runs on one GPU (n > 2^32: 64-bit offsets), 5b is the output stress case
('a'^(2^30), 'a'^16: occ = n - 15).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="3,4,5a,5b")
ap.add_argument("--patterns", type=int, default=40, help="patterns per (config, m)")
ap.add_argument("--reps", type=int, default=2, help="timed repetitions (best is reported)")
ap.add_argument("--no-index", dest="index", action="store_false",
                help="text kernels only (no equality-mask index)")
a = ap.parse_args()
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
result = {}
for cfg in a.configs.split(","):
    for w in synth.config_workloads(cfg):
        text = synth.text_torch(w.spec, 0, w.n, device=dev)
        # the text's equality-mask index over the values its qualifying searches need (built
        # once per text, timed separately: its cost is shared by every search of the text)
        ix, build_us = None, 0.0
        if a.index:
            allp = [epsm.plan(p) for m in w.ms
                    for p in synth.extract_patterns_torch(text, w.start_seed(m), m,
                                                          min(a.patterns, w.patterns_per_m))[0]]
            vals = epsm.index_values(allp)
            for p in allp:
                p.close()
            if vals:
                ix = epsm.EqIndex()
                ix.build_async(text, vals, stream=stream)      # (allocates the planes: not timed)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                ix.build_async(text, vals, stream=stream)
                e1.record(stream)
                torch.cuda.synchronize()
                build_us = e0.elapsed_time(e1) * 1e3
                result[f"{w.name}/index_build"] = {"us": round(build_us, 1), "values": len(vals)}
                print(f"{w.name}: index of {len(vals)} values built in {build_us:.1f} us", file=sys.stderr)
        for m in w.ms:
            count = min(a.patterns, w.patterns_per_m)
            pats, _ = synth.extract_patterns_torch(text, w.start_seed(m), m, count)
            plans = [epsm.plan(p) for p in pats]
            occ = torch.zeros(len(plans), dtype=torch.int64, device=dev)
            epsm.search_batch_async(plans, text, occ, stream=stream)        # counts -> buffer sizes
            torch.cuda.synchronize()
            cap = int(occ.max().item()) + 1
            nbuf = min(len(plans), 80)
            free = torch.cuda.mem_get_info(dev)[0]
            nbuf = max(1, min(nbuf, int(0.8 * free) // (8 * cap)))
            pool = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(nbuf)]
            outs = [pool[j % nbuf] for j in range(len(plans))]
            best = None
            for _ in range(a.reps + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                epsm.search_batch_async(plans, text, occ, outs=outs, stream=stream, index=ix)
                e1.record(stream)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) * 1e-3 / len(plans)
                best = t if best is None or t < best else best
            o = occ.cpu().tolist()
            alg = sum(w.n + 8 * x for x in o) / len(o)
            result[f"{w.name}/m={m}"] = {
                "us_per_search": round(best * 1e6, 2), "text_GBps": round(w.n / best / 1e9, 1),
                "alg_GBps": round(alg / best / 1e9, 1), "patterns": len(plans),
                "occ_total": int(sum(o)), "note": "buffers shared" if nbuf < len(plans) else ""}
            print(f"{w.name} m={m:2d}: {best * 1e6:9.2f} us/search  {w.n / best / 1e9:7.1f} GB/s text"
                  f"  {alg / best / 1e9:7.1f} GB/s alg  occ_total={sum(o)}", file=sys.stderr, flush=True)
            del pool, outs
            for p in plans:
                p.close()
        if ix is not None:
            ix.close()
        del text
        torch.cuda.empty_cache()
print(json.dumps(result))
