"""Oracle parity of the bench's exact launch configuration at full size.

bench.py times BASELINE.json configs[1]: 256 MiB texts over sigma symbols, 100 patterns per
(sigma, m) extracted from the text, run through the batch API (persistent launches of up to
40 searches) over the text's equality-mask index.  At that size every CTA of an index launch
walks hundreds of chunks (40 searches x 2048 chunks over 148 CTAs), so the multi-chunk
bookkeeping of the index variants (tiles per stage, parking-slot reuse, job-slot switching)
runs exactly as in the timed region.  The oracle cannot scan 40 x 256 MiB per group, so:

  * exact window parity: every search's GPU positions inside the first, the last and three
    random 1 MiB windows equal the oracle over that window (+ m - 1 bytes);
  * the full count of two patterns per group against oracle_count (the whole text);
  * properties of every search at any size: strictly increasing, inside [0, n - m], every
    reported position verifies against the pattern, the extraction start is reported.

Bar: bit-exact (Sec. 1: all occurrences).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N = 256 * synth.MiB
W = 1 << 20
K = 40                      # searches per launch (the kernel's maximum, as in the bench)


@pytest.fixture(scope="module")
def epsm():
    import paper_1209_6449_b200 as e
    return e


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda:0")


def window_parity(pos_dev, text_host, pattern, a, w=W):
    n = text_host.size
    m = len(pattern)
    b = min(n, a + w + m - 1)
    want = oracle.search(pattern, text_host[a:b]) + np.uint64(a)
    lo, hi = torch.searchsorted(pos_dev, torch.tensor([a, a + w], device=pos_dev.device)).tolist()
    got = pos_dev[lo:hi].cpu().numpy().astype(np.uint64)
    got = got[got <= np.uint64(b - m)]
    assert np.array_equal(got, want), (pattern, a, got[:5], want[:5])


def verify_all(pos, text_dev, pattern):
    """Every reported position verifies (t[s + j] = p[j] for all j): one gather per j."""
    p = torch.as_tensor(np.frombuffer(pattern, np.uint8).copy(), device=text_dev.device)
    for j in range(len(pattern)):
        assert bool((text_dev[pos + j] == p[j]).all()), (pattern, j)


@pytest.mark.parametrize("sigma", [2, 4, 8, 256])
def test_index_batch_at_bench_scale(epsm, dev, sigma):
    spec = synth.raw_sigma_spec(sigma, (2, sigma))
    text = synth.text_torch(spec, 0, N, device=dev)
    host = text.cpu().numpy()
    rng = np.random.default_rng(1000 + sigma)
    groups = {}
    for m in (2, 4, 8, 16):
        pats, starts = synth.extract_patterns_torch(text, (2, sigma, m), m, K)
        groups[m] = ([epsm.plan(p) for p in pats], pats, starts)
    allplans = [pl for g in groups.values() for pl in g[0]]
    with epsm.eq_index(text, epsm.index_values(allplans)) as ix:
        for m, (plans, pats, starts) in groups.items():
            occ_c = torch.zeros(K, dtype=torch.int64, device=dev)
            epsm.count_batch_async(plans, text, occ_c)          # count kernel: sizes the outputs
            torch.cuda.synchronize()
            caps = occ_c.cpu().tolist()
            outs = [torch.empty(max(c, 1), dtype=torch.int64, device=dev) for c in caps]
            occ = torch.full((K,), -1, dtype=torch.int64, device=dev)
            epsm.search_batch_async(plans, text, occ, outs=outs, index=ix)
            torch.cuda.synchronize()
            occ = occ.cpu().tolist()
            n_ix = sum(len(pl.index_values()) > 0 for pl in plans)
            if m <= 8:
                assert n_ix == K, (sigma, m, n_ix)                # the index variants ran
            for j in range(K):
                assert occ[j] == caps[j], (sigma, m, j)
                pos = outs[j][: occ[j]]
                if occ[j] > 1:
                    assert bool((pos[1:] > pos[:-1]).all()), (sigma, m, j)
                if occ[j]:
                    assert int(pos[0]) >= 0 and int(pos[-1]) <= N - m
                assert bool((pos == int(starts[j])).any()), (sigma, m, j)   # recall
                verify_all(pos, text, pats[j])                               # precision
                for a in [0, N - W] + rng.integers(0, N - W, size=3).tolist():
                    window_parity(pos, host, pats[j], int(a))
            for j in (0, K - 1):
                assert occ[j] == oracle.count(pats[j], host), (sigma, m, j)
            del outs
    for pl in allplans:
        pl.close()


@pytest.mark.parametrize("sigma", [2, 4, 8, 16, 64, 128, 256])
def test_group_search_at_bench_scale(epsm, dev, sigma):
    """The bench's step as it runs: per (sigma, m) ONE group call over the 256 MiB text with its
    100 extracted patterns, the index over the dense patterns' bytes -- every path at full size:
    the shared sampled / code-mode passes (thousands of chunks per CTA, lists and re-filtered
    chunks), the dense patterns one by one or in the mask pass, the duplicates' copies.  Checks:
    the oracle's full count of two searches per group, window parity of every distinct pattern
    (first, last, two random 1 MiB windows), the per-search properties (ascending, in range,
    every position verifies, the extraction start reported), duplicates equal."""
    spec = synth.raw_sigma_spec(sigma, (2, sigma))
    text = synth.text_torch(spec, 0, N, device=dev)
    host = text.cpu().numpy()
    rng = np.random.default_rng(2000 + sigma)
    P = 100
    groups = {}
    for m in (2, 4, 8, 16, 32):
        pats, starts = synth.extract_patterns_torch(text, (2, sigma, m), m, P)
        groups[m] = (epsm.group(pats), pats, starts)
    vals = sorted({v for g, _, _ in groups.values() for v in g.index_values()})
    ix = epsm.eq_index(text, bytes(vals)) if vals else None
    for m, (g, pats, starts) in groups.items():
        occ_c = torch.zeros(P, dtype=torch.int64, device=dev)
        g.count_async(text, occ_c, index=ix)
        torch.cuda.synchronize()
        caps = occ_c.cpu().tolist()
        outs = [torch.empty(max(c, 1), dtype=torch.int64, device=dev) for c in caps]
        occ = torch.full((P,), -1, dtype=torch.int64, device=dev)
        g.search_async(text, occ, outs=outs, index=ix)
        torch.cuda.synchronize()
        occ = occ.cpu().tolist()
        assert occ == caps, (sigma, m)
        first = {}
        for j in range(P):
            pos = outs[j][: occ[j]]
            if pats[j] in first:                                          # a duplicate: equal
                assert torch.equal(pos, outs[first[pats[j]]][: occ[j]]), (sigma, m, j)
                continue
            first[pats[j]] = j
            if occ[j] > 1:
                assert bool((pos[1:] > pos[:-1]).all()), (sigma, m, j)
            assert int(pos[0]) >= 0 and int(pos[-1]) <= N - m
            assert bool((pos == int(starts[j])).any()), (sigma, m, j)    # recall
            verify_all(pos, text, pats[j])                                # precision
            for a in [0, N - W] + rng.integers(0, N - W, size=2).tolist():
                window_parity(pos, host, pats[j], int(a))
        for j in (0, P - 1):
            assert occ[j] == oracle.count(pats[j], host), (sigma, m, j)
        del outs
        g.close()
    if ix is not None:
        ix.close()
