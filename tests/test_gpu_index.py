"""GPU parity of the equality-mask index path (epsm_eqidx_* + epsm_search_batch_index_async).

The index holds EPSMa's equality masks of a whole text, one bit plane per
byte value; searches with at most 8 distinct bytes stream their planes instead of the text
and run the shift-AND on them.  Bar: bit-exact positions and counts against the CPU oracle,
on texts spanning several tiles/chunks with ragged tails, planted occurrences at every
slice/tile/chunk boundary, texts shorter than one 64-position word, patterns whose bytes are
missing from the index or exceed 8 distinct values (text kernels), and misuse errors.
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

TILE = 32768
CHUNK = 4 * TILE


@pytest.fixture(scope="module")
def epsm():
    import paper_1209_6449_b200 as e
    return e


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda:0")


def run_batch(epsm, pats, td, index, caps=None):
    plans = [epsm.plan(p) for p in pats]
    n = td.numel()
    outs = [torch.empty(max(n, 1), dtype=torch.int64, device=td.device) for _ in pats]
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=td.device)
    epsm.search_batch_async(plans, td, occ, outs=outs, caps=caps, index=index)
    torch.cuda.synchronize()
    res = []
    for j in range(len(pats)):
        k = int(occ[j])
        c = k if caps is None else min(k, caps[j])
        res.append((k, outs[j][:c].cpu().numpy().astype(np.uint64)))
    for p in plans:
        p.close()
    return res


def assert_parity(pats, res, t, label, caps=None):
    for j, (p, (k, got)) in enumerate(zip(pats, res)):
        want = oracle.search(p, t)
        assert k == want.size, (label, j, len(p), k, want.size)
        c = want.size if caps is None else min(want.size, caps[j])
        assert np.array_equal(got, want[:c]), (label, j, len(p))


def planted_text(rng, n, sigma, pats):
    t = rng.integers(0, sigma, size=n, dtype=np.uint8)
    edges = []
    for b in range(0, n, 64):          # every lane segment boundary of the first chunk,
        if b > CHUNK:
            break
        edges.append(b)
    edges += list(range(TILE, n, TILE)) + list(range(CHUNK, n, CHUNK)) + [n]
    for i, e in enumerate(edges):
        p = pats[i % len(pats)]
        m = len(p)
        for s in (e - m, e - m // 2, e - 1):   # windows ending at, straddling, starting at e
            if 0 <= s and s + m <= n:
                t[s:s + m] = np.frombuffer(p, dtype=np.uint8)
    return t


@pytest.mark.parametrize("sigma", [2, 4, 8, 16])
def test_index_batch_matches_oracle(epsm, dev, sigma):
    rng = np.random.default_rng(1000 + sigma)
    n = 2 * CHUNK + 3 * TILE + 777
    seed_t = rng.integers(0, sigma, size=n, dtype=np.uint8)
    pats = []
    for m in (1, 2, 3, 4, 5, 7, 8, 9, 12, 16, 17, 24, 31, 32):
        for _ in range(2):
            s0 = int(rng.integers(0, n - m + 1))
            pats.append(seed_t[s0:s0 + m].tobytes())
    t = planted_text(rng, n, sigma, pats)
    td = torch.from_numpy(t).to(dev)
    vals = epsm.index_values(pats)
    assert len(vals) > 0
    with epsm.eq_index(td, vals) as ix:
        assert set(ix.values) == set(vals)
        res = run_batch(epsm, pats, td, ix)
        # the count kernel over the same index
        plans = [epsm.plan(p) for p in pats]
        occ = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
        for _ in range(2):
            epsm.count_batch_async(plans, td, occ, index=ix)
        torch.cuda.synchronize()
        assert occ.cpu().tolist() == [k for k, _ in res]
    assert_parity(pats, res, t, f"sigma={sigma}")


def test_index_dense_and_truncated(epsm, dev):
    """'a'^n and period-2 texts: every start (or every other) matches; caps truncate."""
    for n in (1, 63, 64, 65, 1000, TILE + 1, CHUNK + 64 * 3 + 5):
        ta = np.full(n, ord("a"), dtype=np.uint8)
        tb = np.frombuffer((b"ab" * (n // 2 + 1))[:n], dtype=np.uint8).copy()
        for t in (ta, tb):
            td = torch.from_numpy(t).to(dev)
            pats = [p for p in (b"a", b"aa", b"ab", b"ba", b"a" * 9, b"ab" * 16, b"b") if len(p) <= n]
            caps = [max(0, n // 3) if j % 2 else n for j in range(len(pats))]
            with epsm.eq_index(td, b"ab") as ix:
                res = run_batch(epsm, pats, td, ix, caps=caps)
            assert_parity(pats, res, t, f"dense n={n}", caps=caps)


def test_index_mixed_eligibility(epsm, dev):
    """Searches whose bytes are missing from the index, or with more than 8 distinct bytes,
    or longer than 32, take the text kernels inside the same batch call."""
    rng = np.random.default_rng(77)
    n = CHUNK + 2 * TILE + 13
    t = rng.integers(0, 12, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    pats = []
    for m in (2, 4, 8, 10, 16, 20, 32, 40):
        for _ in range(3):
            s0 = int(rng.integers(0, n - m + 1))
            pats.append(t[s0:s0 + m].tobytes())
    with epsm.eq_index(td, bytes(range(6))) as ix:     # only values 0..5
        res = run_batch(epsm, pats, td, ix)
    assert_parity(pats, res, t, "mixed")


def test_index_rebuild_and_reuse(epsm, dev):
    """One index object rebuilt over texts of growing size (re-allocation) and reused by
    several batches; searching a text the index was not built over is an error."""
    rng = np.random.default_rng(5)
    ix = epsm.EqIndex()
    try:
        for n in (500, 3 * TILE + 5, 2 * CHUNK + 1):
            t = rng.integers(0, 3, size=n, dtype=np.uint8)
            td = torch.from_numpy(t).to(dev)
            ix.build_async(td, b"\x00\x01\x02")
            pats = [t[s:s + m].tobytes() for m in (2, 6, 11, 32) for s in (0, n // 2, n - m)]
            for _ in range(2):
                res = run_batch(epsm, pats, td, ix)
                assert_parity(pats, res, t, f"rebuild n={n}")
        other = torch.from_numpy(rng.integers(0, 3, size=n, dtype=np.uint8)).to(dev)
        plans = [epsm.plan(b"\x00\x01")]
        occ = torch.zeros(1, dtype=torch.int64, device=dev)
        with pytest.raises(epsm.EpsmError):
            epsm.search_batch_async(plans, other, occ, index=ix)
    finally:
        ix.close()


def test_index_build_errors(epsm, dev):
    buf = torch.zeros(1000, dtype=torch.uint8, device=dev)
    ix = epsm.EqIndex()
    try:
        with pytest.raises(epsm.EpsmError) as e:
            ix.build_async(buf[1:], b"\x00")            # not 16-byte aligned
        assert e.value.code == epsm.EPSM_EALIGN
        with pytest.raises(epsm.EpsmError) as e:
            ix.build_async(buf, b"\x00\x00")            # duplicate value
        assert e.value.code == epsm.EPSM_EINVAL
        with pytest.raises(epsm.EpsmError):
            ix.build_async(buf, bytes(range(256)) + b"\x00")   # more than 256 planes (and a duplicate)
        with pytest.raises(epsm.EpsmError):
            ix.build_async(buf, b"")
    finally:
        ix.close()


def test_index_many_values(epsm, dev):
    """64 planes (the maximum): a 64-letter text, short patterns over it, plane ids above 32;
    and an index over values that do not occur (their planes are all zero)."""
    rng = np.random.default_rng(64)
    n = CHUNK + 5 * TILE + 3
    t = rng.integers(0, 64, size=n, dtype=np.uint8)
    pats = [t[s:s + m].tobytes() for m in (1, 2, 3, 4, 6, 8, 12, 16) for s in rng.integers(0, n - m, 4)]
    pats += [bytes([63, 62]), bytes([200, 201]), bytes([0, 63, 0])]
    t = planted_text(rng, n, 64, pats)
    td = torch.from_numpy(t).to(dev)
    vals = bytes(range(63, -1, -1))                # reversed: plane id != value
    with epsm.eq_index(td, vals) as ix:
        assert ix.values == vals
        res = run_batch(epsm, pats, td, ix)
    assert_parity(pats, res, t, "64 planes")
    with epsm.eq_index(td, bytes(range(100, 164))) as ix:   # none of these bytes occur
        res = run_batch(epsm, [bytes([100, 101]), bytes([100]) * 5], td, ix)
    assert all(k == 0 for k, _ in res)


def test_index_all_256_values(epsm, dev):
    """Every byte value has a plane (bit-sliced build); short patterns over a 256-letter text,
    including bytes 0x00 and 0xFF and a ragged tail."""
    rng = np.random.default_rng(256)
    n = 3 * TILE + 4321
    t = rng.integers(0, 256, size=n, dtype=np.uint8)
    pats = [t[s:s + m].tobytes() for m in (1, 2, 3, 4, 8) for s in rng.integers(0, n - m, 5)]
    pats += [b"\x00\xff", b"\xff\x00", b"\x00" * 3, t[n - 4:].tobytes()]
    t = planted_text(rng, n, 256, pats)
    td = torch.from_numpy(t).to(dev)
    with epsm.eq_index(td, bytes(range(256))) as ix:
        assert ix.values == bytes(range(256))
        res = run_batch(epsm, pats, td, ix)
    assert_parity(pats, res, t, "256 planes")


def test_index_empty_and_short_texts(epsm, dev):
    """n = 0 and n < m over an index: no occurrence, occ written as 0."""
    buf = torch.zeros(64, dtype=torch.uint8, device=dev)
    for n in (0, 1, 3):
        td = buf[:n]
        plans = [epsm.plan(p) for p in (b"\x00", b"\x00\x00", b"\x00\x00\x00\x00", b"\x01\x00")]
        occ = torch.full((len(plans),), -1, dtype=torch.int64, device=dev)
        outs = [torch.empty(4, dtype=torch.int64, device=dev) for _ in plans]
        with epsm.eq_index(td, b"\x00\x01") as ix:
            epsm.search_batch_async(plans, td, occ, outs=outs, index=ix)
            torch.cuda.synchronize()
        want = [max(0, n - len(p.pattern) + 1) if set(p.pattern) == {0} else 0 for p in plans]
        assert occ.cpu().tolist() == want, (n, occ.cpu().tolist())
        for j, w in enumerate(want):
            assert outs[j][:w].cpu().tolist() == list(range(w))


def test_index_on_another_stream(epsm, dev):
    """Build and searches ordered on a side stream (the index is stream-ordered like the rest)."""
    rng = np.random.default_rng(9)
    n = CHUNK + 777
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    pats = [t[s:s + m].tobytes() for m in (2, 4, 8) for s in (5, n // 3)]
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    plans = [epsm.plan(p) for p in pats]
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
    outs = [torch.empty(n, dtype=torch.int64, device=dev) for _ in pats]
    ix = epsm.EqIndex()
    try:
        ix.build_async(td, epsm.index_values(plans), stream=side)
        epsm.search_batch_async(plans, td, occ, outs=outs, stream=side, index=ix)
        side.synchronize()
        for j, p in enumerate(pats):
            want = oracle.search(p, t)
            assert int(occ[j]) == want.size
            assert np.array_equal(outs[j][:want.size].cpu().numpy().astype(np.uint64), want)
    finally:
        ix.close()
