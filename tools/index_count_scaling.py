"""Count-over-index time per search vs batch size (diagnostic)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1209_6449_b200 as epsm  # noqa: E402
import synth  # noqa: E402

dev = torch.device('cuda:0')
n = 256 * synth.MiB
t = synth.text_torch(synth.raw_sigma_spec(32, (2, 32)), 0, n, device=dev)
pats, _ = synth.extract_patterns_torch(t, (2, 32, 2), 2, 16)
plans = [epsm.plan(p) for p in pats]
ix = epsm.eq_index(t, epsm.index_values(plans))
occ = torch.zeros(16, dtype=torch.int64, device=dev)
for k in (1, 2, 4, 16):
    best = 1e9
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        epsm.count_batch_async(plans[:k], t, occ, index=ix)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / k)
    print(f"k={k:2d}: {best:.1f} us per count search over the index")
same = [plans[0]] * 16
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    epsm.count_batch_async(same, t, occ, index=ix)
    e1.record()
    torch.cuda.synchronize()
print(f"16 x the same pattern (same planes, L2-hot): {e0.elapsed_time(e1) * 1e3 / 16:.1f} us per search")
