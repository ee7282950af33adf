"""The paper's EPSM on the host (cpu_epsm/, SSE4.2) against the oracle.

cpu_epsm is a second host baseline, not the oracle: it follows Fig. 1 -- EPSMa's
wscmp shift-AND for m < 4, EPSMb's mpsadbw wsmatch + wsblend filter for 4 <= m < 32, EPSMc's
CRC block fingerprints every (floor(m/16) - 1) * 16 bytes for m >= 32 -- and every procedure
must return exactly Occ(p, t).  Cases: every dispatch class, texts whose
length is not a multiple of 16 (the partial last block, the missing blend partner), periodic
texts (dense overlapping occurrences, EPSMc's fingerprint lists with many offsets), occurrences
planted at both text ends, caps below occ, n < m.
"""
import numpy as np
import pytest

import cpu_epsm
import oracle


def _check(p, t):
    want = oracle.search(p, t)
    got = cpu_epsm.search(p, t)
    assert got.dtype == np.uint64
    assert np.array_equal(got, want), (bytes(p)[:8], len(p), t.size, got[:8], want[:8])
    assert cpu_epsm.count(p, t) == want.size


def test_dispatch_classes():
    assert [cpu_epsm.variant(m) for m in (1, 3, 4, 16, 31, 32, 100)] == list("aabbbcc")


@pytest.mark.parametrize("sigma", [2, 4, 20, 256])
def test_random_all_lengths(sigma):
    rng = np.random.default_rng(sigma)
    for m in list(range(1, 40)) + [47, 48, 63, 64, 65, 100, 130, 257]:
        for n in (0, 1, m - 1, m, m + 1, 15, 16, 17, 31, 33, 1000, 4099):
            if n < 0:
                continue
            t = rng.integers(0, sigma, size=n, dtype=np.uint8)
            pats = []
            if n >= m:
                for s in (0, n - m, int(rng.integers(0, n - m + 1))):
                    pats.append(t[s:s + m].copy())
            pats.append(rng.integers(0, sigma, size=m, dtype=np.uint8))
            for p in pats:
                _check(p, t)


@pytest.mark.parametrize("period", [1, 2, 3, 5, 16, 17])
def test_periodic_dense(period):
    rng = np.random.default_rng(period)
    u = rng.integers(0, 256, size=period, dtype=np.uint8)
    t = np.tile(u, 5000 // period + 2)[:5003]
    for m in (1, 2, 3, 4, 7, 8, 9, 15, 16, 17, 31, 32, 33, 48, 64, 96):
        p = t[7:7 + m].copy()
        _check(p, t)


def test_all_starts_each_block_phase():
    # an occurrence at every phase 0..15 of a 16-byte block, for each class
    rng = np.random.default_rng(7)
    for m in (2, 3, 5, 8, 12, 20, 32, 40, 64):
        t = rng.integers(0, 4, size=3000, dtype=np.uint8)
        p = rng.integers(4, 8, size=m, dtype=np.uint8)     # symbols absent from the text
        for ph in range(16):
            s = 160 + 37 * ph
            s = s - (s % 16) + ph
            t[s:s + m] = p
        t[:m] = p
        t[-m:] = p
        _check(p, t)


def test_cap_and_empty():
    t = np.full(1000, 97, dtype=np.uint8)
    got = cpu_epsm.search(b"aa", t, cap=5)
    assert list(got) == [0, 1, 2, 3, 4]
    assert cpu_epsm.count(b"aa", t) == 999
    assert cpu_epsm.search(b"a" * 40, t[:39]).size == 0
    with pytest.raises(ValueError):
        cpu_epsm.count(b"", t)


def test_many_threads():
    rng = np.random.default_rng(3)
    t = rng.integers(0, 4, size=200_000, dtype=np.uint8)
    pats = [t[s:s + m].copy() for m, s in zip((2, 6, 20, 40), (5, 900, 70_000, 150_000))]
    for p, got in zip(pats, cpu_epsm.search_many(pats, t, threads=4)):
        assert np.array_equal(got, oracle.search(p, t))
