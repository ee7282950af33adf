"""Host logic of the group search (no GPU needed: epsm_group_create does no device work).

Deduplication (identical patterns share one pass and one result), the split into passes of
at most 255 distinct patterns, the sampled geometry the cost model picks (every window of
length m must hold exactly one sample: SK + q - 1 <= m, and the table must hold the D * SK
grams), the set_geometry test hook, and argument errors.
"""
import numpy as np
import pytest

import paper_1209_6449_b200 as epsm


def test_dedup_and_info():
    g = epsm.group([b"ab", b"cd", b"ab", b"ab"]).set_dense(0)
    info = g.info()
    assert info["m"] == 2 and info["k"] == 4 and info["distinct"] == 2 and len(info["passes"]) == 1
    assert info["dense"] == 0
    g.close()


def test_dense_split():
    # sigma = 2: every 2-gram is estimated at 1/4 per byte -> all dense (searched one by one);
    # sigma = 256, m = 8: none dense; set_dense moves the threshold, set_geometry forces all
    rng = np.random.default_rng(1)
    t2 = rng.integers(0, 2, size=1 << 14, dtype=np.uint8)
    pats = [t2[s:s + 2].tobytes() for s in rng.integers(0, t2.size - 2, size=50)]
    info = epsm.group(pats).info()
    assert info["dense"] == info["distinct"] and info["passes"] == []
    t8 = rng.integers(0, 256, size=1 << 14, dtype=np.uint8)
    pats8 = [t8[s:s + 8].tobytes() for s in rng.integers(0, t8.size - 8, size=50)]
    assert epsm.group(pats8).info()["dense"] == 0
    # leave-one-out byte frequencies: each pattern's bytes among the other 3 patterns are 1/2 each
    g = epsm.group([b"\x00\x01", b"\x01\x00", b"\x00\x00", b"\x01\x01"] * 2)
    assert g.set_dense(0).info()["dense"] == 0
    assert g.set_dense(1).info()["dense"] == 0          # 1/4 < 1/2
    assert g.set_dense(3).info()["dense"] == g.info()["distinct"]
    g.set_geometry(2, 1)
    assert g.info()["dense"] == 0 and len(g.info()["passes"]) == 1
    with pytest.raises(epsm.EpsmError):
        g.set_dense(65)
    g.close()


@pytest.mark.parametrize("sigma", [2, 4, 20, 256])
def test_geometry_is_valid(sigma):
    rng = np.random.default_rng(sigma)
    t = rng.integers(0, sigma, size=1 << 16, dtype=np.uint8)
    for m in range(1, 33):
        for k in (1, 7, 100):
            pats = [t[s:s + m].tobytes() for s in rng.integers(0, t.size - m, size=k)]
            info = epsm.group(pats).set_dense(0).info()
            assert info["distinct"] == len(set(pats))
            for q, sk in info["passes"]:
                if sk == 0:                                      # code mode (auto: the table, <= 14 bits)
                    cb = max(1, (len(set(b"".join(pats))) - 1).bit_length())
                    assert q == m and m * cb <= 14, (m, cb)
                    continue
                assert 1 <= q <= min(m, 16) and sk in (1, 2, 4, 8, 16)
                assert sk + q - 1 <= m, (m, q, sk)               # one sample per window
                assert sk * min(255, info["distinct"]) <= 4096


def test_large_alphabet_long_patterns_sample_sparsely():
    rng = np.random.default_rng(3)
    pats = [rng.integers(0, 256, size=32, dtype=np.uint8).tobytes() for _ in range(100)]
    (q, sk), = epsm.group(pats).set_dense(0).info()["passes"]
    assert sk == 16                       # one lookup per 16 text bytes (EPSMc's stride idea)


def test_passes_split_at_255_distinct():
    pats = [i.to_bytes(2, "little") for i in range(600)] + [b"\x00\x00"] * 5
    info = epsm.group(pats).set_dense(0).info()
    assert info["distinct"] == 600 and len(info["passes"]) == 3


def test_set_geometry_validation():
    g = epsm.group([b"abcdefgh"] * 3)
    g.set_geometry(4, 4)
    assert g.info()["passes"] == [(4, 4)]
    for q, sk in ((0, 1), (9, 1), (4, 3), (4, 8), (17, 1), (8, 32)):
        with pytest.raises(epsm.EpsmError) as ei:
            g.set_geometry(q, sk)
        assert ei.value.code == epsm.EPSM_EINVAL
    with pytest.raises(epsm.EpsmError):                       # 8 symbols x 8 bytes: 24 key bits
        g.set_geometry(8, 0)
    g.close()
    g = epsm.group([b"abababab", b"bbbbaaaa"])
    g.set_geometry(8, 0)                                      # the code mode (2 symbols: 8 key bits)
    assert g.info()["passes"] == [(8, 0)]
    g.close()
    g = epsm.group([bytes(range(i, i + 16)) for i in range(0, 64, 16)])
    with pytest.raises(epsm.EpsmError):                       # 64 symbols x 16 bytes: no code mode
        g.set_geometry(16, 0)
    g.close()


def test_create_errors():
    with pytest.raises(ValueError):
        epsm.group([b"ab", b"abc"])
    with pytest.raises(ValueError):
        epsm.group([])
    with pytest.raises(epsm.EpsmError) as ei:
        epsm.group([b"x" * 33])
    assert ei.value.code == epsm.EPSM_EUNSUP
    with pytest.raises(epsm.EpsmError) as ei:
        epsm.group([b"ab"] * 1025)
    assert ei.value.code == epsm.EPSM_EUNSUP
