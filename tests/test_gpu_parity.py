"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: bit-exact positions and counts (integer/index work).  Sizes span several
32 KiB tiles (and 128 KiB look-back chunks) with ragged tails; every unit/tile alignment is hit by rotating the
text's base address; edge cases cover n < m, n = 0, m = 1 and 32, dense output,
cap truncation and misaligned text pointers.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TILE = 32768          # bytes per TMA stage (kTile)
CHUNK = 4 * TILE      # look-back chunk (kChunkTiles tiles)
SLICE = 2048          # text bytes one consumer warp covers per tile
SEG = 64              # text bytes one consumer lane covers per tile


@pytest.fixture(scope="module")
def epsm():
    import paper_1209_6449_b200 as e
    return e


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda:0")


def gpu_search(epsm, pattern, text_dev, cap=None):
    pos, occ = epsm.search(pattern, text_dev, cap=cap)
    return pos.cpu().numpy().astype(np.uint64), occ


def check(epsm, pattern, text_np, text_dev, label=""):
    got, occ = gpu_search(epsm, pattern, text_dev)
    want = oracle.search(pattern, text_np)
    assert occ == want.size, (label, pattern, occ, want.size)
    if not np.array_equal(got, want):
        bad = np.flatnonzero(got[: min(got.size, want.size)] != want[: min(got.size, want.size)])
        raise AssertionError(f"{label} m={len(pattern)} first mismatch at index {bad[:5]}")
    return occ


def test_paper_wsmatch_figure_on_gpu(epsm, dev):
    """b = [1010,0111,1010] occurs in a at {1, 5}."""
    a = bytes([0b0110, 0b1010, 0b0111, 0b1010, 0b0100, 0b1010, 0b0111, 0b1010, 0b0000, 0b1010, 0b0100, 0b0010])
    b = bytes([0b1010, 0b0111, 0b1010])
    t = torch.tensor(list(a), dtype=torch.uint8, device=dev)
    got, occ = gpu_search(epsm, b, t)
    assert got.tolist() == [1, 5] and occ == 2


def test_exhaustive_binary_concatenated_all_alignments(epsm, dev):
    """Every binary pattern of length 1..12 against every binary text of length <= 10
    (joined by 0x02 separators), at every base-address rotation mod 16."""
    pieces = [b"\x02"]
    for n in range(1, 11):
        for bits in itertools.product(b"\x00\x01", repeat=n):
            pieces.append(bytes(bits))
            pieces.append(b"\x02")
    big = np.frombuffer(b"".join(pieces), dtype=np.uint8)
    buf = torch.zeros(big.size + 64, dtype=torch.uint8, device=dev)
    pats = [bytes(b) for m in range(1, 13) for b in itertools.product(b"\x00\x01", repeat=m)]
    rng = np.random.default_rng(3)
    for rot in range(16):
        buf[rot:rot + big.size] = torch.from_numpy(big).to(dev)
        t = buf[rot:rot + big.size]
        sel = pats if rot in (0, 5) else [pats[i] for i in rng.choice(len(pats), 300, replace=False)]
        for p in sel:
            got, occ = gpu_search(epsm, p, t)
            want = oracle.search(p, big)
            assert occ == want.size and np.array_equal(got, want), (rot, p)


@pytest.mark.parametrize("sigma", [2, 4, 20, 27, 64, 256])
def test_random_fuzz_with_planted_boundaries(epsm, dev, sigma):
    rng = np.random.default_rng(100 + sigma)
    sizes = [0, 1, 15, 16, 17, 31, 33, 1000, TILE - 1, TILE, TILE + 1, 3 * TILE + 777, 5 * TILE + 31]
    for n in sizes:
        t = rng.integers(0, sigma, size=n, dtype=np.uint8)
        for m in (1, 2, 3, 4, 5, 7, 8, 9, 12, 15, 16, 17, 24, 31, 32):
            if n >= m and rng.random() < 0.8:
                p = rng.integers(0, sigma, size=m, dtype=np.uint8)
                # plant at 0, n-m, unit and tile edges (s = -1, 0 mod 16 and mod TILE)
                for s in {0, n - m, 15, 16, TILE - 1, TILE, TILE - m + 1, 2 * TILE - 3}:
                    if 0 <= s <= n - m:
                        t[s:s + m] = p
                p = p.tobytes()
            else:
                p = rng.integers(0, sigma, size=m, dtype=np.uint8).tobytes()
            td = torch.from_numpy(t.copy()).to(dev)
            check(epsm, p, t, td, label=f"sigma={sigma} n={n}")


@pytest.mark.parametrize("offset", [1, 3, 7, 8, 13, 15])
def test_misaligned_text_pointer(epsm, dev, offset):
    rng = np.random.default_rng(offset)
    full = rng.integers(0, 4, size=3 * TILE + 100, dtype=np.uint8)
    fd = torch.from_numpy(full).to(dev)
    t = full[offset: offset + 2 * TILE + 41]
    td = fd[offset: offset + 2 * TILE + 41]
    for m in (1, 2, 4, 6, 11, 32):
        p = t[TILE - 2: TILE - 2 + m].tobytes()
        check(epsm, p, t, td, label=f"offset={offset}")


def test_dense_unary_closed_form(epsm, dev):
    """'a'^m in 'a'^n: positions are exactly 0..n-m (dense output, many staging rounds)."""
    n = 3 * TILE + 123
    td = torch.full((n,), ord("a"), dtype=torch.uint8, device=dev)
    for m in (1, 2, 4, 5, 16, 17, 32):
        pos, occ = epsm.search(b"a" * m, td)
        assert occ == n - m + 1
        assert torch.equal(pos, torch.arange(n - m + 1, device=dev, dtype=torch.int64))
        assert epsm.count(b"a" * m, td) == n - m + 1


def test_periodic_text(epsm, dev):
    u = b"ACGTTGCA"
    t = np.frombuffer(u * 5000, dtype=np.uint8)
    td = torch.from_numpy(t.copy()).to(dev)
    for c in range(len(u)):
        for m in (8, 9, 16, 31):
            p = (u * 10)[c:c + m]
            got, occ = gpu_search(epsm, p, td)
            assert got.tolist() == list(range(c, t.size - m + 1, len(u)))


def test_cap_truncation_and_count(epsm, dev):
    rng = np.random.default_rng(11)
    t = rng.integers(0, 2, size=4 * TILE + 5, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    p = bytes([0, 1, 1])
    want = oracle.search(p, t)
    for cap in (0, 1, 7, 1000, want.size - 1, want.size, want.size + 10):
        got, occ = gpu_search(epsm, p, td, cap=cap)
        assert occ == want.size
        assert np.array_equal(got, want[:cap])
    assert epsm.count(p, td) == want.size


def test_edge_cases(epsm, dev):
    td = torch.tensor([1, 2, 3], dtype=torch.uint8, device=dev)
    assert gpu_search(epsm, b"\x01\x02\x03\x04", td)[1] == 0        # m > n
    assert gpu_search(epsm, b"\x01\x02\x03", td)[0].tolist() == [0]  # p = t
    empty = torch.empty(0, dtype=torch.uint8, device=dev)
    assert gpu_search(epsm, b"\x01", empty)[1] == 0
    assert epsm.count(b"\x01", empty) == 0
    with pytest.raises(epsm.EpsmError):
        epsm.plan(b"")
    with pytest.raises(epsm.EpsmError) as ei:
        epsm.plan(b"x" * (epsm.MAX_M_LONG + 1))
    assert ei.value.code == epsm.EPSM_EUNSUP


def test_nul_pattern_never_matches_padding(epsm, dev):
    """Zero bytes are symbols; the kernel's zero-filled staging past the text end
    must never produce a match."""
    for n in (1, 5, 16, 17, TILE + 3):
        t = np.zeros(n, dtype=np.uint8)
        td = torch.from_numpy(t).to(dev)
        for m in (1, 2, 4, 8, 32):
            check(epsm, b"\x00" * m, t, td, label=f"nul n={n}")


def test_async_and_host_apis(epsm, dev):
    rng = np.random.default_rng(5)
    t = rng.integers(0, 4, size=5 * TILE + 9, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    p = t[1000:1006].tobytes()
    want = oracle.search(p, t)
    pl = epsm.plan(p)
    out = torch.empty(want.size + 5, dtype=torch.int64, device=dev)
    occ_d = torch.zeros(1, dtype=torch.int64, device=dev)
    for _ in range(3):   # plan reuse: epochs advance, status words never leak across calls
        epsm.search_async(pl, td, out, occ_d)
        torch.cuda.synchronize()
        assert int(occ_d.item()) == want.size
        assert np.array_equal(out[: want.size].cpu().numpy().astype(np.uint64), want)
    epsm.count_async(pl, td, occ_d)
    assert int(occ_d.item()) == want.size
    hout = np.zeros(want.size, dtype=np.uint64)
    occ = epsm.search_host(pl, t, hout)
    assert occ == want.size and np.array_equal(hout, want)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_emulated_shards_compose(epsm, dev, world):
    """Production ownership/halo rules, shards scanned one after another on one GPU."""
    from paper_1209_6449_b200 import sharding
    rng = np.random.default_rng(world)
    n = 7 * TILE + 1234
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    for m in (2, 8, 32):
        p = t[500:500 + m].copy()
        for r in range(1, world):                       # straddle every cut
            b = sharding.shard_base(n, world, r)
            s = max(0, b - m // 2)
            if s + m <= n:
                t[s:s + m] = p
        td = torch.from_numpy(t).to(dev)
        pl = epsm.plan(p.tobytes())
        run = sharding.local_search_cuda(pl)
        parts, total = [], 0
        for r in range(world):
            base, owned, slen = sharding.shard_layout(n, world, r)
            pos, occ = run(td[base:base + slen], owned, base, n)
            parts.append(pos.cpu().numpy().astype(np.uint64))
            total += occ
        want = oracle.search(p.tobytes(), t)
        assert total == want.size
        assert np.array_equal(np.concatenate(parts), want)


def test_launch_counter_moves(epsm, dev):
    td = torch.zeros(100, dtype=torch.uint8, device=dev)
    before = epsm.launch_count()
    epsm.search(b"\x00\x00", td)
    assert epsm.launch_count() > before


def test_plan_reuse_many_chunks(epsm, dev):
    """One plan, many launches over a text of many chunks (> one CTA per SM): the chunk-id
    counter bookkeeping and the status epochs must carry over launches exactly."""
    rng = np.random.default_rng(77)
    n = 300 * 128 * 1024 + 12345           # ~300 chunks of 128 KiB
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    p = t[5000:5006].tobytes()
    want = oracle.search(p, t)
    pl = epsm.plan(p)
    out = torch.empty(want.size + 8, dtype=torch.int64, device=dev)
    occ_d = torch.zeros(1, dtype=torch.int64, device=dev)
    for i in range(5):
        epsm.search_async(pl, td, out, occ_d)
        epsm.count_async(pl, td, occ_d[0:1] if i % 2 else occ_d)
    torch.cuda.synchronize()
    assert int(occ_d.item()) == want.size
    for _ in range(3):
        pos, occ = epsm.search(pl, td, out=out)
        assert occ == want.size and np.array_equal(pos.cpu().numpy().astype(np.uint64), want)
        assert epsm.count(pl, td) == want.size


def _edges(n, m):
    """Starts that put a window across every kind of internal boundary of the kernel: the
    lane segment (64 B), the warp slice (2 KiB), the tile (32 KiB) and the chunk (128 KiB)."""
    out = set()
    for unit in (SEG, SLICE, TILE, CHUNK):
        for k in (1, 2, 3, 5):
            e = k * unit
            for d in (-m, -m + 1, -1, 0, 1):
                s = e + d
                if 0 <= s <= n - m:
                    out.add(s)
    out.update({0, n - m})
    return sorted(out)


@pytest.mark.parametrize("sigma", [2, 4, 256])
def test_internal_boundaries_multi_chunk(epsm, dev, sigma):
    """Occurrences planted across lane-segment, slice, tile and chunk edges of a text of
    several chunks with a ragged tail, for packed (m <= 8) and sampled (m >= 9) filters."""
    rng = np.random.default_rng(900 + sigma)
    n = 5 * CHUNK + 3 * TILE + 777
    base = rng.integers(0, sigma, size=n, dtype=np.uint8)
    for m in (2, 3, 4, 8, 9, 12, 13, 16, 20, 24, 28, 31, 32):
        t = base.copy()
        p = rng.integers(0, sigma, size=m, dtype=np.uint8)
        for s in _edges(n, m):
            t[s:s + m] = p
        td = torch.from_numpy(t).to(dev)
        occ = check(epsm, p.tobytes(), t, td, label=f"edges sigma={sigma}")
        assert epsm.count(p.tobytes(), td) == occ


def test_sampled_filter_repeated_and_periodic_grams(epsm, dev):
    """Patterns whose q-grams repeat (one table bucket holding several candidate offsets)
    and periodic texts where every sample hits: the sampled filter's candidate masks."""
    rng = np.random.default_rng(4242)
    n = 2 * CHUNK + 12345
    for m in (9, 11, 12, 15, 16, 17, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32):
        for unit in (b"a", b"ab", b"abc", b"abcd", b"aab", b"abcdefgh"):
            p = (unit * 40)[:m]
            t = np.frombuffer((unit * (n // len(unit) + 1))[:n], dtype=np.uint8).copy()
            # sprinkle mismatches so that some windows fail late in the verification
            t[rng.integers(0, n, size=200)] = ord("z")
            td = torch.from_numpy(t).to(dev)
            check(epsm, p, t, td, label=f"periodic unit={unit!r}")


def _gram_hash(words):
    """Test-side copy of the kernel's gram fingerprint (a multiply-add over little-endian
    words, kernel epsm_kernels.cuh gram_hash); used only to BUILD adversarial inputs."""
    mul = (0x9E3779B1, 0x85EBCA77, 0xC2B2AE3D, 0x27D4EB2F)
    h = 0
    for i, w in enumerate(words):
        h = (h + w * mul[i]) & 0xFFFFFFFF
    return h


def test_sampled_filter_bucket_collisions(epsm, dev):
    """Grams of one pattern that share a table bucket with different fingerprints make the
    bucket a wildcard; text grams that share a bucket (and even the fingerprint) with a
    pattern gram but differ must be rejected by the naive check.  Inputs are searched for
    with the kernel's hash so both cases really occur."""
    rng = np.random.default_rng(99)
    m = 32                      # sampled (SK, SQ) = (16, 16): grams p[i .. i+15], i = 1..16
    found = None
    for _ in range(4000):
        p = rng.integers(0, 256, size=m, dtype=np.uint8)
        hs = [_gram_hash(np.frombuffer(p[i:i + 16].tobytes(), dtype="<u4").tolist()) for i in range(1, 17)]
        idx = [h >> 21 for h in hs]
        if len(set(idx)) < len(idx):
            found = p
            break
    assert found is not None
    p = found
    # text: the pattern planted, plus decoys that share each gram's bucket index but differ
    n = CHUNK + 999
    t = rng.integers(0, 256, size=n, dtype=np.uint8)
    for s in (0, 100, SEG - 3, SLICE - 17, TILE - 20, n - m):
        t[s:s + m] = p
    decoy = p.copy()
    decoy[20] ^= 0x40            # a near miss that still matches the first 16 bytes of some grams
    for s in (5000, 9000, TILE + 5):
        t[s:s + m] = decoy
    td = torch.from_numpy(t).to(dev)
    check(epsm, p.tobytes(), t, td, label="bucket collisions")


@pytest.mark.parametrize("sigma", [2, 4, 256])
def test_long_patterns(epsm, dev, sigma):
    """m > 32 (EPSMc's block fingerprints, checked against device memory):
    planted occurrences across internal boundaries and at the text end, ragged sizes."""
    rng = np.random.default_rng(5000 + sigma)
    for n in (100, 5000, 2 * CHUNK + 4321):
        base = rng.integers(0, sigma, size=n, dtype=np.uint8)
        for m in (33, 34, 35, 40, 47, 48, 63, 64, 65, 100, 257, 1000, 4096):
            if m > n:
                continue
            t = base.copy()
            p = rng.integers(0, sigma, size=m, dtype=np.uint8)
            for s in _edges(n, m)[::3]:
                t[s:s + m] = p
            td = torch.from_numpy(t).to(dev)
            occ = check(epsm, p.tobytes(), t, td, label=f"long sigma={sigma} n={n}")
            assert epsm.count(p.tobytes(), td) == occ


def test_long_patterns_dense_and_misaligned(epsm, dev):
    """'a'^m in 'a'^n for m > 32 (every start verifies the whole window) and a misaligned
    text whose last byte ends a match (reads stay inside the last 16-byte block)."""
    n = CHUNK + 77
    td = torch.full((n,), ord("a"), dtype=torch.uint8, device=dev)
    for m in (33, 64, 300):
        pos, occ = epsm.search(b"a" * m, td)
        assert occ == n - m + 1
        assert torch.equal(pos, torch.arange(n - m + 1, device=dev, dtype=torch.int64))
    rng = np.random.default_rng(8)
    full = rng.integers(0, 256, size=TILE + 200, dtype=np.uint8)
    fd = torch.from_numpy(full).to(dev)
    for off in (1, 5, 11):
        t = full[off:off + TILE + 101]
        p = t[-70:].tobytes()
        check(epsm, p, t, fd[off:off + TILE + 101], label=f"long misaligned off={off}")


def test_batch_search_many_patterns_one_text(epsm, dev):
    """epsm_search_batch_async: k searches over one text in persistent launches (runs of equal
    m, at most 40 per launch) -- every search's positions and occ equal the oracle's, with
    per-search caps (truncation), count-only searches and patterns absent from the text."""
    rng = np.random.default_rng(31337)
    n = 3 * CHUNK + 5 * TILE + 99
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    pats = []
    for m in [2] * 3 + [5] * 4 + [8] * 45 + [16] * 5 + [32] * 3 + [40] * 2 + [4] * 2:
        s0 = int(rng.integers(0, n - m + 1))
        p = t[s0:s0 + m].tobytes() if rng.random() < 0.8 else bytes([7]) * m   # 7 never occurs
        pats.append(p)
    plans = [epsm.plan(p) for p in pats]
    wants = [oracle.search(p, t) for p in pats]
    caps = [w.size if j % 5 else max(0, w.size - 3) for j, w in enumerate(wants)]
    outs = [torch.empty(max(c, 1), dtype=torch.int64, device=dev) for c in caps]
    occ = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
    before = epsm.launch_count()
    epsm.search_batch_async(plans, td, occ, outs=outs, caps=caps)
    torch.cuda.synchronize()
    launches = epsm.launch_count() - before
    # one launch per run of <= 40 searches of one kernel variant (m and filter)
    assert launches <= 3 * len({len(p) for p in pats}), launches
    occ_h = occ.cpu().numpy()
    for j, (w, c) in enumerate(zip(wants, caps)):
        assert occ_h[j] == w.size, (j, len(pats[j]))
        got = outs[j][:min(c, w.size)].cpu().numpy().astype(np.uint64)
        assert np.array_equal(got, w[:c]), (j, len(pats[j]))
    # count only (no outputs), twice on the same stream (workspace parity alternation)
    occ2 = torch.zeros(len(pats), dtype=torch.int64, device=dev)
    for _ in range(2):
        epsm.search_batch_async(plans, td, occ2)
    torch.cuda.synchronize()
    assert np.array_equal(occ2.cpu().numpy(), np.array([w.size for w in wants]))
    # the count kernel, batched (per-search counters in the workspace, published by the last CTA)
    occ3 = torch.full((len(pats),), -1, dtype=torch.int64, device=dev)
    for _ in range(2):
        epsm.count_batch_async(plans, td, occ3)
    torch.cuda.synchronize()
    assert np.array_equal(occ3.cpu().numpy(), np.array([w.size for w in wants]))


def test_batch_dense_and_small_texts(epsm, dev):
    """Batches on texts smaller than one chunk (fewer chunks than CTAs, several searches per
    CTA) and dense outputs ('a'^n): ordering across the searches' chunk ranges."""
    for n in (10, 1000, TILE + 7, CHUNK - 1):
        td = torch.full((n,), ord("a"), dtype=torch.uint8, device=dev)
        pats = [b"a" * m for m in (2, 2, 2, 2)] + [b"a" * 9] * 3 + [b"ab", b"ba"]
        pats = [p for p in pats if len(p) <= n]
        plans = [epsm.plan(p) for p in pats]
        outs = [torch.empty(n, dtype=torch.int64, device=dev) for _ in pats]
        occ = torch.zeros(len(pats), dtype=torch.int64, device=dev)
        epsm.search_batch_async(plans, td, occ, outs=outs)
        torch.cuda.synchronize()
        for j, p in enumerate(pats):
            k = n - len(p) + 1 if set(p) == {ord("a")} else 0
            assert int(occ[j]) == k
            assert torch.equal(outs[j][:k], torch.arange(k, device=dev, dtype=torch.int64))


def test_concurrent_streams_have_separate_workspaces(epsm, dev):
    """Searches enqueued on two streams at once (each stream owns a scan workspace) and
    interleaved single/batch/count launches on one stream (workspace parity alternation)."""
    rng = np.random.default_rng(2024)
    n = 2 * CHUNK + 333
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    pats = [t[s:s + m].tobytes() for s, m in ((100, 3), (5000, 8), (70000, 16), (123, 33))]
    wants = [oracle.search(p, t) for p in pats]
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    results = []
    torch.cuda.synchronize()
    for rep in range(3):
        for si, st in enumerate(streams):
            with torch.cuda.stream(st):
                for j, p in enumerate(pats):
                    pl = epsm.plan(p)
                    out = torch.empty(wants[j].size + 4, dtype=torch.int64, device=dev)
                    occ = torch.zeros(1, dtype=torch.int64, device=dev)
                    if (rep + si + j) % 3 == 0:
                        epsm.search_batch_async([pl], td, occ, outs=[out], stream=st)
                    else:
                        epsm.search_async(pl, td, out, occ, stream=st)
                    occ2 = torch.zeros(1, dtype=torch.int64, device=dev)
                    epsm.count_async(pl, td, occ2, stream=st)
                    results.append((j, out, occ, occ2, pl))
    torch.cuda.synchronize()
    for j, out, occ, occ2, _ in results:
        assert int(occ.item()) == wants[j].size and int(occ2.item()) == wants[j].size
        assert np.array_equal(out[: wants[j].size].cpu().numpy().astype(np.uint64), wants[j])


def test_debug_trace_is_off_by_default(epsm, dev):
    td = torch.zeros(1000, dtype=torch.uint8, device=dev)
    epsm.search(b"\x00\x01", td)
    tr = epsm.debug_trace()
    assert tr.size == 0 or tr.shape[1:] == (1024, 8)


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_shards_batch_compose(epsm, dev, world):
    """Sharded batch (bench N > 1 path) emulated on one GPU: each shard's
    epsm_search_range_batch_async output, placed at the exclusive prefix of the per-shard
    counts, is every search's Occ."""
    from paper_1209_6449_b200 import sharding
    rng = np.random.default_rng(77 + world)
    n = 5 * CHUNK + 4567
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    pats = []
    for m in (2, 4, 8, 9, 16, 24, 32):
        p = t[1000 * m:1000 * m + m].copy()
        for r in range(1, world):
            b = sharding.shard_base(n, world, r)
            t[b - m // 2:b - m // 2 + m] = p
        pats.append(p.tobytes())
    td = torch.from_numpy(t).to(dev)
    plans = [epsm.plan(p) for p in pats]
    wants = [oracle.search(p, t) for p in pats]
    parts = [[] for _ in pats]
    for use_index in (False, True):
        parts = [[] for _ in pats]
        for r in range(world):
            base, owned, slen = sharding.shard_layout(n, world, r)
            occ = torch.zeros(len(pats), dtype=torch.int64, device=dev)
            outs = [torch.empty(w.size + 1, dtype=torch.int64, device=dev) for w in wants]
            # each rank's shard in its own (aligned) buffer, as make_texts builds it
            shard = td[base:base + slen].clone()
            ix = epsm.eq_index(shard, epsm.index_values(plans)) if use_index else None
            epsm.search_range_batch_async(plans, shard, owned, base, n, occ, outs=outs, index=ix)
            torch.cuda.synchronize()
            for j in range(len(pats)):
                k = int(occ[j])
                parts[j].append(outs[j][:k].cpu().numpy().astype(np.uint64))
        for j, w in enumerate(wants):
            assert np.array_equal(np.concatenate(parts[j]), w), (use_index, len(pats[j]))


def test_range_calls_reject_a_short_overlap(epsm, dev):
    """A shard that cannot hold every owned window (shard_len < owned + m - 1 while the text
    goes on) is an error, not a silent drop of the occurrences at the cut."""
    n_total = 10_000
    shard = torch.zeros(1000 + 31, dtype=torch.uint8, device=dev)
    occ = torch.zeros(1, dtype=torch.int64, device=dev)
    out = torch.empty(64, dtype=torch.int64, device=dev)
    long_pl = epsm.plan(b"\x00" * 40)                  # needs 39 halo bytes, the shard has 31
    with pytest.raises(epsm.EpsmError) as ei:
        epsm.search_range_async(long_pl, shard, 1000, 0, n_total, out, occ)
    assert ei.value.code == epsm.EPSM_EINVAL
    with pytest.raises(epsm.EpsmError) as ei:
        epsm.search_range_batch_async([long_pl], shard, 1000, 0, n_total, occ)
    assert ei.value.code == epsm.EPSM_EINVAL
    # the same shard at the end of the text (no bytes beyond it) is fine
    epsm.search_range_async(long_pl, shard, 1000, n_total - 1031, n_total, out, occ)
    torch.cuda.synchronize()
    assert int(occ[0]) == 1031 - 40 + 1
    # m <= 32 fits the 31-byte halo
    epsm.search_range_batch_async([epsm.plan(b"\x00" * 32)], shard, 1000, 0, n_total, occ)
    torch.cuda.synchronize()
    assert int(occ[0]) == 1000


@pytest.mark.parametrize("m", [64, 144, 207, 208, 209, 256, 1000, 4096])
def test_long_stride_path(epsm, dev, m):
    """m >= 64: EPSMc's sampling stride (one 16-byte block every (floor(m/16) - 1) * 16 bytes,
    PAPER.md:600-601) -- planted occurrences at every phase relative to the sampled blocks and
    at both ends, periodic texts (many candidates per block), the batch API with caps and
    count-only searches, shards with an (m-1)-byte halo, misaligned texts."""
    from paper_1209_6449_b200 import sharding
    rng = np.random.default_rng(7000 + m)
    L = 16 * (m // 16 - 1)
    n = max(40 * m, 3 * 2048 * L // 8 + 777)
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    p = rng.integers(0, 4, size=m, dtype=np.uint8)
    step = (m // L + 2) * L                                   # planted windows never overlap
    starts = [0, n - m] + [(j + 1) * step + ph for j, ph in enumerate((0, 1, 15, 16, L - 1, L // 2))
                           if (j + 1) * step + ph + m <= n - m]
    for s in starts:
        t[s:s + m] = p
    td = torch.from_numpy(t).to(dev)
    want = oracle.search(p.tobytes(), t)
    assert set(starts) <= set(want.tolist())
    check(epsm, p.tobytes(), t, td, label=f"stride m={m}")
    assert epsm.count(p.tobytes(), td) == want.size
    # periodic: every start matches a^m-like patterns with period 3
    per = np.tile(np.array([1, 2, 3], np.uint8), n // 3 + 1)[:n]
    check(epsm, per[5:5 + m].tobytes(), per, torch.from_numpy(per).to(dev), label=f"stride periodic m={m}")
    # batch API: caps, count-only, an absent pattern, the same pattern twice
    plans = [epsm.plan(p.tobytes()), epsm.plan(p.tobytes()), epsm.plan(bytes(9 for _ in range(m)))]
    occ = torch.zeros(3, dtype=torch.int64, device=dev)
    outs = [torch.full((want.size + 2,), -1, dtype=torch.int64, device=dev) for _ in range(3)]
    epsm.search_batch_async(plans, td, occ, outs=outs, caps=[want.size + 2, 3, 5])
    torch.cuda.synchronize()
    assert occ.tolist() == [want.size, want.size, 0]
    assert np.array_equal(outs[0][:want.size].cpu().numpy().astype(np.uint64), want)
    assert np.array_equal(outs[1][:3].cpu().numpy().astype(np.uint64), want[:3]) and int(outs[1][3]) == -1
    # shards with an (m-1)-byte halo
    parts = []
    for r in range(3):
        base, owned, slen = sharding.shard_layout(n, 3, r, halo=m - 1)
        o = torch.zeros(1, dtype=torch.int64, device=dev)
        out = torch.empty(want.size + 1, dtype=torch.int64, device=dev)
        epsm.search_range_async(plans[0], td[base:base + slen].clone(), owned, base, n, out, o)
        torch.cuda.synchronize()
        parts.append(out[:int(o)].cpu().numpy().astype(np.uint64))
    assert np.array_equal(np.concatenate(parts), want)
    # misaligned views
    for off in (1, 7):
        check(epsm, p.tobytes(), t[off:], td[off:], label=f"stride misaligned m={m} off={off}")
    for pl in plans:
        pl.close()
