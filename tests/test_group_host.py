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
    g = epsm.group([b"ab", b"cd", b"ab", b"ab"])
    info = g.info()
    assert info["m"] == 2 and info["k"] == 4 and info["distinct"] == 2 and len(info["passes"]) == 1
    g.close()


@pytest.mark.parametrize("sigma", [2, 4, 20, 256])
def test_geometry_is_valid(sigma):
    rng = np.random.default_rng(sigma)
    t = rng.integers(0, sigma, size=1 << 16, dtype=np.uint8)
    for m in range(1, 33):
        for k in (1, 7, 100):
            pats = [t[s:s + m].tobytes() for s in rng.integers(0, t.size - m, size=k)]
            info = epsm.group(pats).info()
            assert info["distinct"] == len(set(pats))
            for q, sk in info["passes"]:
                assert 1 <= q <= min(m, 16) and sk in (1, 2, 4, 8, 16)
                assert sk + q - 1 <= m, (m, q, sk)               # one sample per window
                assert sk * min(255, info["distinct"]) <= 4096


def test_large_alphabet_long_patterns_sample_sparsely():
    rng = np.random.default_rng(3)
    pats = [rng.integers(0, 256, size=32, dtype=np.uint8).tobytes() for _ in range(100)]
    (q, sk), = epsm.group(pats).info()["passes"]
    assert sk == 16                       # one lookup per 16 text bytes (EPSMc's stride idea)


def test_passes_split_at_255_distinct():
    pats = [i.to_bytes(2, "little") for i in range(600)] + [b"\x00\x00"] * 5
    info = epsm.group(pats).info()
    assert info["distinct"] == 600 and len(info["passes"]) == 3


def test_set_geometry_validation():
    g = epsm.group([b"abcdefgh"] * 3)
    g.set_geometry(4, 4)
    assert g.info()["passes"] == [(4, 4)]
    for q, sk in ((0, 1), (9, 1), (4, 3), (4, 8), (17, 1)):
        with pytest.raises(epsm.EpsmError) as ei:
            g.set_geometry(q, sk)
        assert ei.value.code == epsm.EPSM_EINVAL
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
