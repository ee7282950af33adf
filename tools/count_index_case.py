import sys, torch
sys.path.insert(0, '.')
import paper_1209_6449_b200 as epsm, synth
dev = torch.device('cuda:0')
n = 256 * synth.MiB
t = synth.text_torch(synth.raw_sigma_spec(32, (2, 32)), 0, n, device=dev)
pats, _ = synth.extract_patterns_torch(t, (2, 32, 2), 2, 4)
plans = [epsm.plan(p) for p in pats]
ix = epsm.eq_index(t, epsm.index_values(plans))
occ = torch.zeros(4, dtype=torch.int64, device=dev)
for _ in range(3):
    epsm.count_batch_async(plans, t, occ, index=ix)
torch.cuda.synchronize()
print(occ.tolist())
