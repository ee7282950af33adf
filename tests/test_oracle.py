"""Pins for the CPU oracle (oracle/epsm_oracle.c), run with -m "not gpu".

The oracle is the definition Occ(p, t) = {s : 0 <= s <= n-m, t[s..s+m-1] = p}
(Sec. 1) written as a brute force.  These tests pin it to
things other than itself:

* the paper's printed worked figures (tests/golden/);
* CPython's ``bytes.find`` (a different search algorithm) over *every* binary
  text/pattern pair up to length 8, and every binary pattern up to length 12
  against every binary text up to length 12 (concatenated with separators);
* the ``re`` engine (zero-width lookahead, a backtracking matcher) on random
  texts over the paper's alphabet sizes, including NUL bytes;
* closed forms: a^m in a^n has n-m+1 occurrences at 0..n-m; for a periodic text
  u^r (u primitive, |u| = q) and a pattern of length m >= q read at phase c, the
  occurrences are exactly the starts s = c (mod q), s <= n-m.

A plausible slip in the oracle (an off-by-one at n-m, a dropped overlap, a
wrong comparison index, a truncation bug) fails at least one of them.
"""
import itertools
import os
import re

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, v = line.split(":", 1)
            out[k.strip()] = v.split()
    return out


def find_all(p: bytes, t: bytes):
    """Every (overlapping) occurrence via CPython's bytes.find."""
    res = []
    i = t.find(p)
    while i != -1:
        res.append(i)
        i = t.find(p, i + 1)
    return res


def re_all(p: bytes, t: bytes):
    """Every (overlapping) occurrence via the re engine's zero-width lookahead."""
    return [mo.start() for mo in re.finditer(b"(?=" + re.escape(p) + b")", t)]


# --------------------------------------------------------------------------
# Paper worked figures
# --------------------------------------------------------------------------

def test_paper_wsmatch_figure():
    """wsmatch(a, b) with k = 3 reports {1, 5}."""
    g = _read_golden("paper_wsmatch_fig.txt")
    text = bytes(int(x, 2) for x in g["text_bits"])
    pat = bytes(int(x, 2) for x in g["pattern_bits"])
    want = [int(x) for x in g["occurrences"]]
    assert len(text) == 12 and len(pat) == 3
    assert oracle.search(pat, text).tolist() == want
    assert oracle.count(pat, text) == len(want)


def test_paper_wscmp_figure_as_naive_checks():
    """r_i = [a_i = b_i] = naive check of b_i at start i of a."""
    g = _read_golden("paper_wscmp_fig.txt")
    a = bytes(int(x, 2) for x in g["a_bits"])
    b = bytes(int(x, 2) for x in g["b_bits"])
    want = {int(x) for x in g["set_positions"]}
    got = {i for i in range(len(a)) if oracle.verify(b[i:i + 1], a, i)}
    assert got == want == {1, 6, 8, 11}


# --------------------------------------------------------------------------
# Exhaustive binary brute force against bytes.find
# --------------------------------------------------------------------------

def _binary_strings(max_len, min_len=0):
    for n in range(min_len, max_len + 1):
        for bits in itertools.product(b"\x00\x01", repeat=n):
            yield bytes(bits)


def test_exhaustive_binary_pairs_up_to_8():
    """Every binary (p, t) with |t| <= 8, 1 <= |p| <= 9 (so m > n is covered)."""
    texts = list(_binary_strings(8))
    pats = list(_binary_strings(9, 1))
    npairs = 0
    for t in texts:
        tn = np.frombuffer(t, dtype=np.uint8)
        for p in pats:
            if len(p) > len(t) + 1:
                continue
            got = oracle.search(p, tn).tolist()
            assert got == find_all(p, t), (p, t)
            npairs += 1
    assert npairs > 100_000


def test_exhaustive_binary_up_to_12_concatenated():
    """Every binary pattern of length 1..12 against every binary text of length
    <= 12.  The texts are joined by a 0x02 separator, which no binary pattern can
    contain, so Occ over the join is the union of the per-text sets."""
    pieces = [b"\x02"]
    for t in _binary_strings(12, 1):
        pieces.append(t)
        pieces.append(b"\x02")
    big = b"".join(pieces)
    bign = np.frombuffer(big, dtype=np.uint8)
    for m in range(1, 13):
        for p in _binary_strings(m, m):
            got = oracle.search(p, bign)
            want = find_all(p, big)
            assert len(got) == len(want), (p,)
            assert np.array_equal(got, np.asarray(want, dtype=np.uint64)), (p,)


# --------------------------------------------------------------------------
# Random texts over the paper's alphabets against the re engine
# --------------------------------------------------------------------------

@pytest.mark.parametrize("sigma", [2, 4, 20, 27, 256])
@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 1000, 100_000])
def test_random_vs_re(sigma, n):
    rng = np.random.default_rng(1000 * sigma + n)
    t = rng.integers(0, sigma, size=n, dtype=np.uint8)
    tb = t.tobytes()
    for m in (1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 40):
        if n >= m and rng.random() < 0.7:
            s0 = int(rng.integers(0, n - m + 1))
            p = tb[s0:s0 + m]                      # extracted: s0 must be found
        else:
            p = rng.integers(0, sigma, size=m, dtype=np.uint8).tobytes()
            s0 = None
        got = oracle.search(p, t).tolist()
        assert got == re_all(p, tb), (sigma, n, m)
        if s0 is not None:
            assert s0 in got


def test_nul_bytes_are_symbols():
    t = b"\x00\x00\x01\x00\x00\x00"
    assert oracle.search(b"\x00\x00", t).tolist() == [0, 3, 4]
    assert oracle.search(b"\x00", t).tolist() == [0, 1, 3, 4, 5]


# --------------------------------------------------------------------------
# Closed forms
# --------------------------------------------------------------------------

def test_unary_closed_form():
    """'a'^m in 'a'^n: exactly n-m+1 occurrences at 0..n-m."""
    for n in range(0, 130):
        t = b"a" * n
        for m in range(1, 40):
            got = oracle.search(b"a" * m, t)
            want = np.arange(max(n - m + 1, 0), dtype=np.uint64)
            assert np.array_equal(got, want), (n, m)


@pytest.mark.parametrize("u", [b"ab", b"ACGT", b"aab", b"abcab" + b"d", b"\x00\x01\x01"])
def test_periodic_closed_form(u):
    """t = u^r (u primitive, q = |u|).  A pattern of length m >= q taken at phase c
    of u^inf occurs exactly at the starts s = c (mod q) with s <= n-m, so
    occ = floor((n-m-c)/q) + 1."""
    q = len(u)
    for r in (1, 2, 5, 37):
        t = u * r
        n = len(t)
        inf = u * (r + 40)
        for c in range(q):
            for m in range(q, min(33, n + 1)):
                p = inf[c:c + m]
                got = oracle.search(p, t).tolist()
                want = list(range(c, n - m + 1, q))
                assert got == want, (u, r, c, m)
                assert len(want) == ((n - m - c) // q + 1 if n - m - c >= 0 else 0)


def test_known_small_cases():
    assert oracle.search(b"aa", b"aaaa").tolist() == [0, 1, 2]
    assert oracle.search(b"ab", b"ab" * 16).tolist() == list(range(0, 32, 2))
    assert oracle.search(b"abc", b"abc").tolist() == [0]          # p = t
    assert oracle.search(b"abcd", b"abc").tolist() == []          # m > n
    assert oracle.search(b"x", b"").tolist() == []                # n = 0


# --------------------------------------------------------------------------
# Argument contract
# --------------------------------------------------------------------------

def test_empty_pattern_is_error():
    with pytest.raises(ValueError):
        oracle.search(b"", b"abc")


def test_cap_truncation_returns_smallest_positions_and_full_count():
    t = b"a" * 100
    pos, occ = oracle.search_capped(b"aa", t, cap=7)
    assert occ == 99
    assert pos.tolist() == list(range(7))
    pos, occ = oracle.search_capped(b"aa", t, cap=0)
    assert occ == 99 and pos.size == 0


def test_verify_range():
    assert oracle.verify(b"ab", b"ab", 0)
    assert not oracle.verify(b"ab", b"ab", 1)      # s > n-m
    assert not oracle.verify(b"ab", b"a", 0)       # n < m


def test_search_many_matches_single():
    rng = np.random.default_rng(7)
    t = rng.integers(0, 4, size=50_000, dtype=np.uint8)
    pats = [t[s:s + m].tobytes() for s, m in [(0, 2), (100, 4), (49_990, 10), (7, 1)]]
    many = oracle.search_many(pats, t, threads=4)
    for p, got in zip(pats, many):
        assert np.array_equal(got, oracle.search(p, t))
    counts = oracle.search_many(pats, t, threads=4, count_only=True)
    assert counts == [len(x) for x in many]
