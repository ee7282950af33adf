import sys, time
import torch
sys.path.insert(0, ".")
import paper_1209_6449_b200 as epsm
import synth
dev = torch.device("cuda:0")
n = 256 * synth.MiB
for s, m in [(256, 32), (64, 16), (256, 4)]:
    t = synth.text_torch(synth.raw_sigma_spec(s, (2, s)), 0, n, device=dev)
    pats, _ = synth.extract_patterns_torch(t, (2, s, m), m, 100)
    g = epsm.group(pats)
    occ = torch.zeros(100, dtype=torch.int64, device=dev)
    g.count_async(t, occ); torch.cuda.synchronize()
    cap = int(occ.max()) + 1
    outs = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(100)]
    for _ in range(3): g.search_async(t, occ, outs=outs)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 20
    a.record(); h0 = time.perf_counter()
    for _ in range(R): g.search_async(t, occ, outs=outs)
    h1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
    print(f"sigma={s} m={m}: host {1e6*(h1-h0)/R:.1f} us/call, gpu {1e3*a.elapsed_time(b)/R:.1f} us/call", flush=True)
    # GPU time with the host out of the way: a long sleep kernel first lets the host enqueue everything
    torch.cuda._sleep(50_000_000)
    a.record()
    for _ in range(R): g.search_async(t, occ, outs=outs)
    b.record(); torch.cuda.synchronize()
    print(f"   queued ahead: gpu {1e3*a.elapsed_time(b)/R:.1f} us/call", flush=True)
