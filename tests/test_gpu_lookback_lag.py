"""A lagging look-back warp (EPSM_FLAGS=4 slows it by ~16 us per chunk): the consumers run
ahead until the parking slots stop them, and every search must still be bit-exact -- the
slots' reuse is guarded (a warp waits for the look-back warp's scan of chunk k before parking
chunk k + 8, and for its prefix before writing chunk k out).  Run in a subprocess: the flags
are read once per process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import numpy as np, torch, oracle, paper_1209_6449_b200 as epsm
rng = np.random.default_rng(8)
n = 8 * (1 << 20) + 12345                   # 64+ chunks per search: > 8 per CTA in a batch
dev = torch.device("cuda:0")
t = rng.integers(0, 256, size=n, dtype=np.uint8)
# 40 patterns, each planted ~2 times per 128 KiB chunk at random places: every chunk has
# positions in a few warps' slices only, different ones from chunk to chunk
pats = [bytes(rng.integers(0, 256, size=8, dtype=np.uint8)) for _ in range(40)]
for p in pats:
    for s in rng.integers(0, n - 8, size=2 * (n >> 17)):
        t[s:s + 8] = np.frombuffer(p, dtype=np.uint8)
pats += [t[s:s + 2].tobytes() for s in (5, 77)]      # and two dense-ish ones
td = torch.from_numpy(t).to(dev)
plans = [epsm.plan(p) for p in pats]
wants = [oracle.search(p, t) for p in pats]
for use_index in (False, True):
    ix = epsm.eq_index(td, epsm.index_values(plans)) if use_index else None
    occ = torch.zeros(len(pats), dtype=torch.int64, device=dev)
    outs = [torch.empty(w.size + 1, dtype=torch.int64, device=dev) for w in wants]
    epsm.search_batch_async(plans, td, occ, outs=outs, index=ix)
    torch.cuda.synchronize()
    for j, w in enumerate(wants):
        assert int(occ[j]) == w.size, (use_index, j)
        assert np.array_equal(outs[j][:w.size].cpu().numpy().astype(np.uint64), w), (use_index, j)
print("ok")
'''


def test_lagging_lookback_warp_stays_exact():
    env = dict(os.environ, EPSM_FLAGS="4", PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
