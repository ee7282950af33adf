"""Debug driver for the group search: one small case per (sigma, m), checked against the oracle
(run under compute-sanitizer on the GPU box)."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1209_6449_b200 as epsm  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
sig = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ms = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4, 8, 16, 32]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3 * 32768 + 77
for m in ms:
    t = rng.integers(0, sig, size=n, dtype=np.uint8)
    pats = [t[s:s + m].tobytes() for s in rng.integers(0, n - m, size=10)]
    g = epsm.group(pats)
    print("m", m, g.info(), flush=True)
    td = torch.from_numpy(t).to(dev)
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
    outs = [torch.zeros(n, dtype=torch.int64, device=dev) for _ in pats]
    g.count_async(td, occ)
    torch.cuda.synchronize()
    print(" count ok", occ.tolist()[:4], flush=True)
    g.search_async(td, occ, outs=outs)
    torch.cuda.synchronize()
    bad = 0
    for j, p in enumerate(pats):
        w = oracle.search(p, t)
        k = int(occ[j])
        got = outs[j][:k].cpu().numpy().astype(np.uint64)
        if k != w.size or not np.array_equal(got, w):
            bad += 1
            print("  MISMATCH", j, k, w.size, got[:6], w[:6])
    print(" search", "ok" if not bad else f"{bad} bad", flush=True)
