"""GPU parity of the group search (epsm_group_*): k patterns of one length in one pass.

Every search of a group must return exactly its own Occ(p_j, t), as the
oracle computes it pattern by pattern.  Cases: every alphabet / pattern length class, every
(gram length, stride) geometry the kernels are compiled for, duplicate and absent patterns,
occurrences planted at every lane (64 B), slice (2 KiB) and chunk (32 KiB) edge and at the text
ends, dense texts whose chunks overflow the per-chunk occurrence lists (positions recomputed
from the text) mixed with sparse chunks (positions from the lists), misaligned text pointers,
capacities below occ, count-only calls, shards, and groups of more than 255 distinct patterns
(several passes).
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


def run_group(epsm, pats, td, caps=None, geom=None, count_only=False, dense=0, index=None):
    """dense=0 (default here): every pattern through the group kernels (the kernels under
    test); dense=None: the library's split (dense patterns one by one, over `index`)."""
    g = epsm.group(pats)
    if dense is not None:
        g.set_dense(dense)
    if geom is not None:
        g.set_geometry(*geom)
    n = td.numel()
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=td.device)
    if count_only:
        g.count_async(td, occ, index=index)
        torch.cuda.synchronize()
        g.close()
        return [(int(o), None) for o in occ.cpu().tolist()]
    outs = [torch.full((max(n, 1),), -7, dtype=torch.int64, device=td.device) for _ in pats]
    g.search_async(td, occ, outs=outs, caps=caps, index=index)
    torch.cuda.synchronize()
    res = []
    for j in range(len(pats)):
        k = int(occ[j])
        c = k if caps is None else min(k, caps[j])
        got = outs[j][:c].cpu().numpy().astype(np.uint64)
        if caps is not None and caps[j] < outs[j].numel():
            assert int(outs[j][caps[j]]) == -7, "wrote past the capacity"
        res.append((k, got))
    g.close()
    return res


def check(pats, res, t, label, caps=None):
    cache = {}
    for j, (p, (k, got)) in enumerate(zip(pats, res)):
        if p not in cache:
            cache[p] = oracle.search(p, t)
        want = cache[p]
        assert k == want.size, (label, j, len(p), k, want.size)
        if got is not None:
            c = want.size if caps is None else min(want.size, caps[j])
            assert np.array_equal(got, want[:c]), (label, j, len(p), got[:8], want[:8])


def planted(rng, n, sigma, m, count, absent=3):
    t = rng.integers(0, sigma, size=n, dtype=np.uint8)
    starts = rng.integers(0, n - m + 1, size=count)
    pats = [t[s:s + m].tobytes() for s in starts]
    # plant the first patterns across lane / slice / chunk edges and at both ends
    edges = [0, n - m]
    for e in (64, 128, 2048, 4096, TILE, 2 * TILE, 3 * TILE + 2048, 4 * TILE - 64):
        for d in (-m + 1, -1, 0):
            if 0 <= e + d <= n - m:
                edges.append(e + d)
    for i, e in enumerate(edges):
        p = np.frombuffer(pats[i % min(len(pats), 5)], np.uint8)
        t[e:e + m] = p
    pats = [t[s:s + m].tobytes() for s in starts]            # (re-read after planting)
    pats += [pats[0], pats[1], pats[0]]                      # duplicates
    pats += [rng.integers(0, 256, size=m, dtype=np.uint8).tobytes() for _ in range(absent)]
    return t, pats


@pytest.mark.parametrize("sigma", [2, 4, 20, 256])
def test_group_alphabets_and_lengths(epsm, dev, sigma):
    rng = np.random.default_rng(sigma)
    n = 5 * TILE + 777
    for m in (1, 2, 3, 4, 5, 7, 8, 9, 12, 16, 17, 20, 24, 31, 32):
        t, pats = planted(rng, n, sigma, m, 30)
        td = torch.from_numpy(t).to(dev)
        check(pats, run_group(epsm, pats, td), t, (sigma, m))


GEOMS = [(q, sk) for q in (1, 2, 3, 4, 5, 7, 8, 9, 12, 13, 16) for sk in (1, 2, 4, 8, 16) if sk + q - 1 <= 32]


@pytest.mark.parametrize("q,sk", GEOMS)
def test_group_every_geometry(epsm, dev, q, sk):
    """Every compiled (key words, stride) variant, forced: same results."""
    rng = np.random.default_rng(100 + 17 * q + sk)
    n = 3 * TILE + 4321
    for sigma, m in ((4, 32), (2, max(17, q + sk - 1)), (256, max(q + sk - 1, 1))):
        t, pats = planted(rng, n, sigma, m, 20)
        td = torch.from_numpy(t).to(dev)
        check(pats, run_group(epsm, pats, td, geom=(q, sk)), t, (q, sk, sigma, m))


def test_group_dense_and_sparse_chunks_mixed(epsm, dev):
    """Chunks over the occurrence-list capacity (positions recomputed from the text) next to
    sparse chunks (positions from the lists) in one launch."""
    rng = np.random.default_rng(5)
    n = 8 * TILE + 99
    t = rng.integers(0, 256, size=n, dtype=np.uint8)
    t[2 * TILE + 100: 5 * TILE - 7] = ord("a")              # dense run over 3 chunks
    t[6 * TILE: 6 * TILE + 3000] = np.tile(np.frombuffer(b"ab", np.uint8), 1500)
    for m in (2, 4, 16, 32):
        pats = [b"a" * m, (b"ab" * 16)[:m], (b"ba" * 16)[:m], b"a" * m,
                t[100:100 + m].tobytes(), t[7 * TILE:7 * TILE + m].tobytes(), b"\x00" * m]
        td = torch.from_numpy(t).to(dev)
        check(pats, run_group(epsm, pats, td), t, ("mixed", m))


def test_group_unary_closed_form(epsm, dev):
    n = 6 * TILE + 13
    td = torch.full((n,), ord("a"), dtype=torch.uint8, device=dev)
    for m in (1, 2, 16, 32):
        pats = [b"a" * m] * 4 + [b"b" * m]
        res = run_group(epsm, pats, td)
        for j in range(4):
            k, got = res[j]
            assert k == n - m + 1 and np.array_equal(got, np.arange(n - m + 1, dtype=np.uint64))
        assert res[4][0] == 0


@pytest.mark.parametrize("offset", [1, 3, 8, 15])
def test_group_misaligned_text(epsm, dev, offset):
    rng = np.random.default_rng(offset)
    n = 2 * TILE + 555
    big = rng.integers(0, 4, size=n + 32, dtype=np.uint8)
    t = big[offset:offset + n]
    bd = torch.from_numpy(big).to(dev)
    td = bd[offset:offset + n]
    for m in (2, 5, 16, 32):
        pats = [t[s:s + m].tobytes() for s in (0, 1, n - m, 12345, 40000)]
        check(pats, run_group(epsm, pats, td), t, ("mis", offset, m))


def test_group_caps_and_counts(epsm, dev):
    rng = np.random.default_rng(9)
    n = 4 * TILE + 1
    t = rng.integers(0, 2, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    pats = [t[s:s + 3].tobytes() for s in (0, 10, 20, 30, 40, 50)]
    occs = [oracle.count(p, t) for p in pats]
    caps = [0, 1, occs[2] // 2, occs[3], occs[4] + 5, 7]
    check(pats, run_group(epsm, pats, td, caps=caps), t, "caps", caps=caps)
    check(pats, run_group(epsm, pats, td, count_only=True), t, "count")


def test_group_short_texts(epsm, dev):
    for n in (0, 1, 2, 15, 16, 17, 31, 32, 33, 64, 65):
        t = np.frombuffer((b"abcabcabca" * 8)[:n], np.uint8).copy()
        td = torch.from_numpy(t).to(dev) if n else torch.empty(0, dtype=torch.uint8, device=dev)
        for m in (1, 2, 3, 16, 32):
            pats = [(b"abc" * 11)[:m], (b"bca" * 11)[:m], b"z" * m]
            check(pats, run_group(epsm, pats, td), t, ("short", n, m))


def test_group_many_distinct_patterns(epsm, dev):
    """More than 255 distinct patterns: several passes, each search still exact."""
    rng = np.random.default_rng(11)
    n = 3 * TILE + 17
    t = rng.integers(0, 256, size=n, dtype=np.uint8)
    starts = rng.integers(0, n - 4, size=700)
    pats = [t[s:s + 4].tobytes() for s in starts] + [b"\x01\x02\x03\x04"] * 3
    g = epsm.group(pats)
    assert len(g.info()["passes"]) >= 3
    g.close()
    check(pats, run_group(epsm, pats, torch.from_numpy(t).to(dev)), t, "many")


@pytest.mark.parametrize("world", [2, 3])
def test_group_shards_compose(epsm, dev, world):
    from paper_1209_6449_b200 import sharding
    rng = np.random.default_rng(50 + world)
    n = 6 * TILE + 345
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    for m in (2, 8, 32):
        pats = [t[s:s + m].tobytes() for s in rng.integers(0, n - m, size=12)]
        for r in range(1, world):                              # straddle every cut
            b = sharding.shard_base(n, world, r)
            t[b - m // 2:b - m // 2 + m] = np.frombuffer(pats[0], np.uint8)
        wants = [oracle.search(p, t) for p in pats]
        td = torch.from_numpy(t).to(dev)
        g = epsm.group(pats)
        parts = [[] for _ in pats]
        for r in range(world):
            base, owned, slen = sharding.shard_layout(n, world, r)
            shard = td[base:base + slen].clone()
            occ = torch.zeros(len(pats), dtype=torch.int64, device=dev)
            outs = [torch.empty(w.size + 1, dtype=torch.int64, device=dev) for w in wants]
            g.search_range_async(shard, owned, base, n, occ, outs=outs)
            torch.cuda.synchronize()
            for j in range(len(pats)):
                parts[j].append(outs[j][:int(occ[j])].cpu().numpy().astype(np.uint64))
        g.close()
        for j, w in enumerate(wants):
            assert np.array_equal(np.concatenate(parts[j]), w), (world, m, j)


@pytest.mark.parametrize("sigma", [2, 4, 16, 256])
@pytest.mark.parametrize("use_index", [False, True])
def test_group_dense_split(epsm, dev, sigma, use_index):
    """The library's split: dense patterns (estimated >= 2^-7 occurrences per byte) searched
    one by one (over the text's index where they qualify), the rest in the shared passes --
    every search still returns its own Occ."""
    rng = np.random.default_rng(200 + sigma)
    n = 9 * TILE + 123
    for m in (2, 4, 8, 16):
        t, pats = planted(rng, n, sigma, m, 40)
        td = torch.from_numpy(t).to(dev)
        g = epsm.group(pats)
        info = g.info()
        g.close()
        if sigma == 2 and m <= 4:
            assert info["dense"] > 0, info
        if sigma == 256 and m >= 4:
            assert info["dense"] == 0, info
        ix = None
        if use_index:
            plans = [epsm.plan(p) for p in set(pats)]
            vals = epsm.index_values(plans)
            ix = epsm.eq_index(td, vals) if vals else None
        check(pats, run_group(epsm, pats, td, dense=None, index=ix), t, ("split", sigma, m, use_index))
        check(pats, run_group(epsm, pats, td, dense=None, index=ix, count_only=True), t, ("split-count", sigma, m))
        if ix is not None:
            ix.close()


def test_group_dense_split_shards(epsm, dev):
    from paper_1209_6449_b200 import sharding
    rng = np.random.default_rng(77)
    n = 7 * TILE + 5
    t = rng.integers(0, 2, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    pats = [t[s:s + 4].tobytes() for s in rng.integers(0, n - 4, size=20)] + [b"\x07" * 4]
    wants = [oracle.search(p, t) for p in pats]
    g = epsm.group(pats)
    assert 0 < g.info()["dense"] < g.info()["distinct"]
    parts = [[] for _ in pats]
    for r in range(2):
        base, owned, slen = sharding.shard_layout(n, 2, r)
        shard = td[base:base + slen].clone()
        ix = epsm.eq_index(shard, b"\x00\x01")
        occ = torch.zeros(len(pats), dtype=torch.int64, device=dev)
        outs = [torch.empty(w.size + 1, dtype=torch.int64, device=dev) for w in wants]
        g.search_range_async(shard, owned, base, n, occ, outs=outs, index=ix)
        torch.cuda.synchronize()
        for j in range(len(pats)):
            parts[j].append(outs[j][:int(occ[j])].cpu().numpy().astype(np.uint64))
        ix.close()
    g.close()
    for j, w in enumerate(wants):
        assert np.array_equal(np.concatenate(parts[j]), w), j


@pytest.mark.parametrize("use_index", [False, True])
def test_group_dense_fanout_phases_and_caps(epsm, dev, use_index):
    """Dense patterns are scanned once and their positions fanned out to every search of the
    pattern: outputs of both 16-byte phases (one job per phase), capacities below occ, a
    count-only slot (no output) -- every search still gets exactly its own Occ."""
    rng = np.random.default_rng(410)
    n = 13 * TILE + 77
    t = rng.integers(0, 2, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    base = [t[s:s + 3].tobytes() for s in (5, 900, 7000)]
    while len(set(base)) < 3:
        base = [bytes(rng.integers(0, 2, size=3, dtype=np.uint8)) for _ in range(3)]
    pats = [base[0]] * 6 + [base[1]] * 5 + [base[2]] * 3
    wants = [oracle.search(p, t) for p in pats]
    g = epsm.group(pats)
    assert g.info()["dense"] == 3
    ix = epsm.eq_index(td, g.index_values()) if use_index and g.index_values() else None
    bufs = [torch.full((w.size + 8,), -4, dtype=torch.int64, device=dev) for w in wants]
    outs = [b[j % 2:] for j, b in enumerate(bufs)]          # alternate 16-byte phases
    caps = [w.size for w in wants]
    caps[1] = wants[1].size // 3
    caps[7] = 5
    outs[4] = None                                           # count only
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
    g.search_async(td, occ, outs=outs, caps=[c if o is not None else 0 for c, o in zip(caps, outs)], index=ix)
    torch.cuda.synchronize()
    for j, w in enumerate(wants):
        assert int(occ[j]) == w.size, j
        if outs[j] is None:
            continue
        c = min(w.size, caps[j])
        got = outs[j][:c].cpu().numpy().astype(np.uint64)
        assert np.array_equal(got, w[:c]), (j, got[:5], w[:5])
        assert int(outs[j][c]) == -4, j                      # nothing past the capacity
    g.close()


@pytest.mark.parametrize("sigma", [2, 3, 4, 16, 100])
def test_group_code_mode(epsm, dev, sigma):
    """The code mode (every start keyed through the patterns' byte codes, exact): forced with
    set_geometry(q, 0) wherever m * ceil(log2(distinct pattern bytes)) <= 16 (<= 14: key table;
    15-16: the wide mode's bitmap + buckets); bytes outside the
    patterns' alphabet break windows; edges, duplicates and absent patterns as elsewhere."""
    rng = np.random.default_rng(500 + sigma)
    n = 7 * TILE + 1001
    for m in (1, 2, 3, 4, 5, 7, 8, 12, 14, 15, 16):
        t, pats = planted(rng, n, sigma, m, 25, absent=2)
        sigp = len(set(b"".join(pats)))
        cb = max(1, (sigp - 1).bit_length())
        td = torch.from_numpy(t).to(dev)
        if m * cb > 16:
            g = epsm.group(pats).set_dense(0)
            with pytest.raises(epsm.EpsmError):
                g.set_geometry(m, 0)
            g.close()
            continue
        check(pats, run_group(epsm, pats, td, geom=(m, 0)), t, ("code", sigma, m))


@pytest.mark.parametrize("m", [1, 2, 3])
def test_group_code_mode_full_slices(epsm, dev, m):
    """Code mode at every start matching (2048 matches per 2 KiB slice: pass 3 ranks the slice
    in two windows of compacted matches) and at about half the starts matching (slices on both
    sides of the window size), with a few distinct patterns per round."""
    n = 5 * TILE + 777
    t = np.tile(np.frombuffer(b"ab", np.uint8), n // 2 + 1)[:n].copy()
    pats = [(b"ab" * 4)[:m], (b"ba" * 4)[:m], b"b" * m, (b"ab" * 4)[:m]]
    td = torch.from_numpy(t).to(dev)
    check(pats, run_group(epsm, pats, td, geom=(m, 0)), t, ("full", m))
    rng = np.random.default_rng(900 + m)
    t = rng.integers(0, 2, size=n, dtype=np.uint8)
    pats = sorted({t[s:s + m].tobytes() for s in range(0, 64)})
    pats += [pats[0]]
    td = torch.from_numpy(t).to(dev)
    check(pats, run_group(epsm, pats, td, geom=(m, 0)), t, ("half", m))


def test_group_code_mode_chosen_for_dense_small_alphabets(epsm):
    rng = np.random.default_rng(7)
    t = rng.integers(0, 2, size=1 << 16, dtype=np.uint8)
    pats = [t[s:s + 8].tobytes() for s in rng.integers(0, t.size - 8, size=100)]
    g = epsm.group(pats).set_dense(5)          # none one by one at 1/256 per byte
    assert g.info()["passes"] == [(8, 0)]
    g.close()


@pytest.mark.parametrize("sigma,m", [(8, 2), (6, 2), (3, 3), (2, 5)])
def test_group_mask_pass(epsm, dev, sigma, m):
    """>= 24 dense patterns over an index: the mask pass (all dense patterns' shift-ANDs over the
    planes in one pass, epsm_mask.cuh) -- every search exact, with duplicates (copied by the
    replicate kernel), capacities, count-only, misaligned outputs and shards."""
    from paper_1209_6449_b200 import sharding
    rng = np.random.default_rng(600 + 10 * sigma + m)
    n = 21 * TILE + 301
    t = rng.integers(0, sigma, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    grams = sorted({t[s:s + m].tobytes() for s in range(0, n - m, 7)})
    pats = grams[:40] + grams[:5] + [bytes([0] * (m - 1) + [200])]      # dups and an absent one
    wants = [oracle.search(p, t) for p in pats]
    g = epsm.group(pats)
    info = g.info()
    assert info["dense"] >= 24, info
    ix = epsm.eq_index(td, g.index_values())
    bufs = [torch.full((w.size + 6,), -2, dtype=torch.int64, device=dev) for w in wants]
    outs = [b[j % 2:] for j, b in enumerate(bufs)]
    caps = [w.size for w in wants]
    caps[3] = wants[3].size // 2
    caps[len(pats) - 2] = 1
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
    g.search_async(td, occ, outs=outs, caps=caps, index=ix)
    torch.cuda.synchronize()
    for j, w in enumerate(wants):
        assert int(occ[j]) == w.size, (j, int(occ[j]), w.size)
        c = min(w.size, caps[j])
        assert np.array_equal(outs[j][:c].cpu().numpy().astype(np.uint64), w[:c]), j
        assert int(outs[j][c]) == -2, j
    occ2 = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
    g.count_async(td, occ2, index=ix)
    torch.cuda.synchronize()
    assert occ2.cpu().tolist() == [w.size for w in wants]
    ix.close()
    # shards, each with its own index
    parts = [[] for _ in pats]
    for r in range(3):
        base, owned, slen = sharding.shard_layout(n, 3, r)
        shard = td[base:base + slen].clone()
        six = epsm.eq_index(shard, g.index_values())
        o = torch.zeros(len(pats), dtype=torch.int64, device=dev)
        so = [torch.empty(w.size + 1, dtype=torch.int64, device=dev) for w in wants]
        g.search_range_async(shard, owned, base, n, o, outs=so, index=six)
        torch.cuda.synchronize()
        for j in range(len(pats)):
            parts[j].append(so[j][:int(o[j])].cpu().numpy().astype(np.uint64))
        six.close()
    for j, w in enumerate(wants):
        assert np.array_equal(np.concatenate(parts[j]), w), ("shard", j)
    g.close()


@pytest.mark.parametrize("dense", [64, 0])
def test_group_many_fanout_sources(epsm, dev, dense):
    """More than 256 duplicated distinct patterns: the multi-source fan-out splits its job table
    into launches of <= 256 sources (dense=64: every pattern scanned one by one and fanned out
    by the batch path; dense=0: the group passes, duplicates fanned out after pass 3), with
    outputs of both 16-byte phases (those sources go through the single-source kernel), odd and
    zero occurrence counts, and capacities below occ."""
    rng = np.random.default_rng(4242 + dense)
    n = 9 * TILE + 333
    t = rng.integers(0, 32, size=n, dtype=np.uint8)
    distinct = sorted({t[s:s + 3].tobytes() for s in range(0, n - 2, 97)})[:300]
    assert len(distinct) == 300
    pats = distinct + distinct[:280] + [bytes([200, 201, 202])] * 2      # (the last: no occurrence)
    wants = {p: oracle.search(p, t) for p in set(pats)}
    g = epsm.group(pats).set_dense(dense)
    bufs = [torch.full((wants[p].size + 8,), -4, dtype=torch.int64, device=dev) for p in pats]
    outs = [b[1:] if j % 7 == 3 else b for j, b in enumerate(bufs)]      # some in the other phase
    caps = [wants[p].size if j % 11 else max(0, wants[p].size - 1) for j, p in enumerate(pats)]
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
    g.search_async(torch.from_numpy(t).to(dev), occ, outs=outs, caps=caps)
    torch.cuda.synchronize()
    for j, p in enumerate(pats):
        w = wants[p]
        assert int(occ[j]) == w.size, j
        c = min(w.size, caps[j])
        assert np.array_equal(outs[j][:c].cpu().numpy().astype(np.uint64), w[:c]), j
        assert int(outs[j][c]) == -4, j
    g.close()


@pytest.mark.parametrize("dense", [0, 64])
def test_ktimer_fanout_bytes(epsm, dev, dense):
    """The benchmark's live timer of the fan-out kernel (epsm_ktimer_*): with every distinct
    pattern asked k times (outputs 16-byte aligned, capacities >= occ), the recorded algorithmic
    bytes are exactly sum over patterns of 8 * occ * k (the source read once, k - 1 copies
    written), occ from the oracle; the records clear on read and nothing is recorded while off."""
    rng = np.random.default_rng(77 + dense)
    n = 11 * TILE + 45
    t = rng.integers(0, 8, size=n, dtype=np.uint8)
    distinct = [t[s:s + 3].tobytes() for s in (5, 900, 4000, 70000)]
    ks = [3, 2, 5, 1]
    pats = [p for p, k in zip(distinct, ks) for _ in range(k)]
    wants = {p: oracle.search(p, t) for p in distinct}
    td = torch.from_numpy(t).to(dev)
    g = epsm.group(pats).set_dense(dense)
    outs = [torch.full((wants[p].size + 8,), -4, dtype=torch.int64, device=dev) for p in pats]
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
    epsm.ktimer_read()
    g.search_async(td, occ, outs=outs)                       # (timer off: not recorded)
    torch.cuda.synchronize()
    assert epsm.ktimer_read() == (0, 0.0, 0.0)
    epsm.ktimer_enable(True)
    try:
        g.search_async(td, occ, outs=outs)
        torch.cuda.synchronize()
    finally:
        epsm.ktimer_enable(False)
    nl, ms, byts = epsm.ktimer_read()
    for j, p in enumerate(pats):
        assert int(occ[j]) == wants[p].size
        assert np.array_equal(outs[j][:wants[p].size].cpu().numpy().astype(np.uint64), wants[p])
    assert nl >= 1 and ms > 0.0
    assert byts == sum(8.0 * wants[p].size * k for p, k in zip(distinct, ks) if k > 1)
    assert epsm.ktimer_read() == (0, 0.0, 0.0)
    g.close()
