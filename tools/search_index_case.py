"""One batched search over an equality-mask index (for ncu): sigma, m, outputs on/off."""
import argparse
import sys
import torch
sys.path.insert(0, '.')
import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sigma", type=int, default=32)
ap.add_argument("--m", type=int, default=2)
ap.add_argument("--k", type=int, default=4)
ap.add_argument("--no-out", action="store_true")
a = ap.parse_args()
dev = torch.device('cuda:0')
n = 256 * synth.MiB
t = synth.text_torch(synth.raw_sigma_spec(a.sigma, (2, a.sigma)), 0, n, device=dev)
pats, _ = synth.extract_patterns_torch(t, (2, a.sigma, a.m), a.m, a.k)
plans = [epsm.plan(p) for p in pats]
ix = epsm.eq_index(t, epsm.index_values(plans))
occ = torch.zeros(a.k, dtype=torch.int64, device=dev)
epsm.search_batch_async(plans, t, occ, index=ix)
torch.cuda.synchronize()
outs = None if a.no_out else [torch.empty(int(occ.max()) + 1, dtype=torch.int64, device=dev) for _ in range(a.k)]
for _ in range(3):
    epsm.search_batch_async(plans, t, occ, outs=outs, index=ix)
torch.cuda.synchronize()
print(occ.tolist())
