"""GPU parity of the group search's code-mode kernels (epsm_code.cuh: per-lane counters, rotated
scan, staged write-out) against the oracle, pattern by pattern (every search
returns exactly its own Occ(p, t), in text order).

The code mode is forced with set_geometry(m, 0); groups of <= 127 distinct patterns of length
<= 8 take the dedicated kernels.  Cases: with and without a spare code (bytes outside the
patterns' alphabet in the text), many chunks per CTA (texts of several hundred chunks), the
largest id (126: the second counter row of every lane), 128 distinct patterns (the general
kernels), misaligned texts, capacities below occ, count-only calls, shards, every start
matching, and matches planted at lane / slice / half-chunk / chunk edges.
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

TILE = 32768


@pytest.fixture(scope="module")
def epsm():
    import paper_1209_6449_b200 as e
    return e


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda:0")


def run(epsm, pats, td, caps=None, count_only=False, code=True):
    g = epsm.group(pats).set_dense(0)
    if code:
        g.set_geometry(len(pats[0]), 0)
    n = td.numel()
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=td.device)
    if count_only:
        g.count_async(td, occ)
        torch.cuda.synchronize()
        g.close()
        return [(int(o), None) for o in occ.cpu().tolist()]
    outs = [torch.full((max(n, 1) + 1,), -7, dtype=torch.int64, device=td.device) for _ in pats]
    g.search_async(td, occ, outs=outs, caps=caps)
    torch.cuda.synchronize()
    res = []
    for j in range(len(pats)):
        k = int(occ[j])
        c = k if caps is None else min(k, caps[j])
        got = outs[j][:c].cpu().numpy().astype(np.uint64)
        assert int(outs[j][c]) == -7, ("wrote past the capacity / occ", j)
        res.append((k, got))
    g.close()
    return res


def check(pats, res, t, label, caps=None):
    cache = {}
    for j, (p, (k, got)) in enumerate(zip(pats, res)):
        if p not in cache:
            cache[p] = oracle.search(p, t)
        want = cache[p]
        assert k == want.size, (label, j, p, k, want.size)
        if got is not None:
            c = want.size if caps is None else min(want.size, caps[j])
            assert np.array_equal(got, want[:c]), (label, j, p, got[:8], want[:8])


def extract(rng, t, m, count, ok=None):
    """count patterns copied from t at random starts (whose bytes all satisfy ok, if given)."""
    pats = []
    while len(pats) < count:
        s = int(rng.integers(0, t.size - m + 1))
        w = t[s:s + m]
        if ok is None or ok(w):
            pats.append(w.tobytes())
    return pats


def plant_edges(t, pats, m):
    """copies of the first patterns across lane, slice, half-chunk and chunk edges and the ends"""
    n = t.size
    edges = [0, n - m]
    for e in (64, 2048, 16384, TILE, TILE + 16384, 3 * TILE, 5 * TILE - 64):
        for d in (-m + 1, -1, 0, 1):
            if 0 <= e + d <= n - m:
                edges.append(e + d)
    for i, e in enumerate(edges):
        t[e:e + m] = np.frombuffer(pats[i % min(len(pats), 4)], np.uint8)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8])
def test_code_alphabet_of_four_with_foreign_bytes(epsm, dev, m):
    """patterns over {0,1,2,3} (cb = 2), text with 3% bytes outside: m <= 4 has a spare code,
    m = 5..7 does not (windows with a foreign byte dropped in the kernel); m = 8 (16 key bits)
    runs the general kernels' wide mode."""
    rng = np.random.default_rng(10 + m)
    n = 6 * TILE + 999
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    foreign = rng.random(n) < 0.03
    t[foreign] = rng.integers(4, 256, size=int(foreign.sum()), dtype=np.uint8)
    pats = extract(rng, t, m, 60, ok=lambda w: bool((w < 4).all()))
    plant_edges(t, pats, m)
    pats = [bytes(p) for p in pats]
    td = torch.from_numpy(t).to(dev)
    check(pats, run(epsm, pats, td), t, ("foreign", m))


@pytest.mark.parametrize("sigma,m", [(2, 8), (4, 4), (16, 2), (2, 5), (8, 3)])
def test_code_many_chunks_per_cta(epsm, dev, sigma, m):
    """bench-like dense groups (100 patterns extracted from a uniform text) over a text of ~600
    chunks: every CTA of both passes loops over several chunks, pass 3 over both halves."""
    rng = np.random.default_rng(100 * sigma + m)
    n = 600 * TILE + 12345
    t = rng.integers(0, sigma, size=n, dtype=np.uint8)
    pats = extract(rng, t, m, 100)
    td = torch.from_numpy(t).to(dev)
    check(pats, run(epsm, pats, td), t, ("bench-like", sigma, m))


def test_code_largest_ids(epsm, dev):
    """127 distinct patterns (ids up to 126: every lane's second counter row) through the
    dedicated kernels, and 128 through the general ones -- the same results."""
    rng = np.random.default_rng(3)
    n = 9 * TILE + 77
    t = rng.integers(0, 16, size=n, dtype=np.uint8)
    allp = sorted({t[s:s + 2].tobytes() for s in range(0, n - 1)})
    rng.shuffle(allp)
    for k in (127, 128):
        pats = allp[:k] + allp[:3]
        check(pats, run(epsm, pats, torch.from_numpy(t).to(dev)), t, ("ids", k))


@pytest.mark.parametrize("offset", [1, 7, 13])
def test_code_misaligned(epsm, dev, offset):
    rng = np.random.default_rng(offset)
    n = 5 * TILE + 333
    base = rng.integers(0, 4, size=n + 32, dtype=np.uint8)
    t = base[offset:offset + n].copy()
    pats = extract(rng, t, 4, 40)
    plant_edges(t, pats, 4)
    base[offset:offset + n] = t
    bd = torch.from_numpy(base).to(dev)
    check(pats, run(epsm, pats, bd[offset:offset + n]), t, ("misaligned", offset))


def test_code_caps_and_count_only(epsm, dev):
    rng = np.random.default_rng(5)
    n = 4 * TILE + 4321
    t = rng.integers(0, 2, size=n, dtype=np.uint8)
    pats = extract(rng, t, 6, 30)
    pats += [pats[0], pats[0], pats[1]]                       # duplicates (fanned out)
    td = torch.from_numpy(t).to(dev)
    want = [oracle.search(p, t).size for p in pats]
    caps = [max(0, w // (2 + j % 3) - j) for j, w in enumerate(want)]
    check(pats, run(epsm, pats, td, caps=caps), t, "caps", caps=caps)
    check(pats, run(epsm, pats, td, count_only=True), t, "count")


def test_code_every_start_and_short_texts(epsm, dev):
    """'ab' repeated: every start matches one of two patterns (runs of 1024 per lane and
    pattern); texts shorter than one lane, one slice, one chunk."""
    for n in (5 * TILE + 17, 3, 63, 64, 65, 2047, 2049, 16385, TILE + 1):
        t = np.tile(np.frombuffer(b"ab", np.uint8), n // 2 + 1)[:n].copy()
        for m in (2, 3, 8):
            if m > n:
                continue
            pats = [(b"ab" * 4)[:m], (b"ba" * 4)[:m], b"a" * m]
            check(pats, run(epsm, pats, torch.from_numpy(t).to(dev)), t, ("every", n, m))


@pytest.mark.parametrize("world", [2, 3])
def test_code_shards_compose(epsm, dev, world):
    """range calls over the shards of sharding.shard_layout (the sharded path's local step):
    positions are global, the union over shards equals the whole text's; a copy of a pattern
    straddles every cut."""
    from paper_1209_6449_b200 import sharding
    rng = np.random.default_rng(9 + world)
    n = 7 * TILE + 555
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    pats = extract(rng, t, 6, 50)
    for r in range(1, world):
        b = sharding.shard_base(n, world, r)
        t[b - 3:b + 3] = np.frombuffer(pats[0], np.uint8)
    td = torch.from_numpy(t).to(dev)
    g = epsm.group(pats).set_dense(0)
    g.set_geometry(6, 0)
    parts = [[] for _ in pats]
    for r in range(world):
        base, owned, slen = sharding.shard_layout(n, world, r)
        shard = td[base:base + slen].clone()
        occ = torch.zeros(len(pats), dtype=torch.int64, device=dev)
        outs = [torch.empty(n, dtype=torch.int64, device=dev) for _ in pats]
        g.search_range_async(shard, owned, base, n, occ, outs=outs)
        torch.cuda.synchronize()
        for j in range(len(pats)):
            parts[j].append(outs[j][:int(occ[j])].cpu().numpy().astype(np.uint64))
    g.close()
    for j, p in enumerate(pats):
        assert np.array_equal(np.concatenate(parts[j]), oracle.search(p, t)), (world, j)
