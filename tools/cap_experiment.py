import sys, torch
sys.path.insert(0, '.')
import paper_1209_6449_b200 as epsm, synth
dev = torch.device('cuda:0')
n = 256 * synth.MiB
for s, m in [(4, 2), (2, 4), (16, 2), (32, 2), (2, 8)]:
    t = synth.text_torch(synth.raw_sigma_spec(s, (2, s)), 0, n, device=dev)
    pats, _ = synth.extract_patterns_torch(t, (2, s, m), m, 16)
    plans = [epsm.plan(p) for p in pats]
    ix = epsm.eq_index(t, epsm.index_values(plans))
    occ = torch.zeros(16, dtype=torch.int64, device=dev)
    epsm.search_batch_async(plans, t, occ, index=ix); torch.cuda.synchronize()
    cap = int(occ.max()) + 1
    outs = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(16)]
    def tm(f):
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / 16)
        return best
    a = tm(lambda: epsm.search_batch_async(plans, t, occ, outs=outs, index=ix))
    b = tm(lambda: epsm.search_batch_async(plans, t, occ, index=ix))
    c = tm(lambda: epsm.search_batch_async(plans, t, occ, outs=outs, caps=[1] * 16, index=ix))
    d = tm(lambda: epsm.count_batch_async(plans, t, occ, index=ix))
    print(f"sigma={s} m={m}: positions {a:.1f} us, no outputs {b:.1f} us, cap 1 {c:.1f} us, "
          f"count kernel {d:.1f} us, occ {int(occ[0])}")
