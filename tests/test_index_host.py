"""Host-side logic of the equality-mask index (no GPU: plans are built on the host).

Which searches of a batch run over an index (epsm_plan_index_values): the pattern's distinct
bytes in order of first occurrence, for m <= 8 with at most 8 distinct bytes, or m <= 31 with
at most 4; everything else keeps the text kernels.  index_values() is the union a batch needs.
Also the C-side argument checks of the index entry points that fail before any device work.
"""
import ctypes

import pytest


@pytest.fixture(scope="module")
def epsm():
    import paper_1209_6449_b200 as e
    return e


@pytest.mark.parametrize("pattern,want", [
    (b"a", b"a"),
    (b"ab", b"ab"),
    (b"abab", b"ab"),
    (b"\x00\xff\x00", b"\x00\xff"),
    (b"baac", b"bac"),                                   # first-occurrence order
    (b"abcdefgh", b"abcdefgh"),                          # m = 8, d = 8
    (b"abcdefghi", b""),                                 # m = 9, d = 9: text kernels
    (b"abcdabcdabcdabcdabcdabcd", b"abcd"),               # m = 24, d = 4
    (b"abcdeabcdeabcdeabcdeabcd", b""),                  # m = 24, d = 5
    (b"ab" * 12 + b"a", b"ab"),                          # m = 25, d = 2
    (b"ab" * 16, b""),                                   # m = 32: text kernels
    (b"aaaaaaaaaaaaaaaa", b"a"),                         # m = 16, d = 1
    (b"x" * 33, b""),                                    # long pattern
])
def test_plan_index_values(epsm, pattern, want):
    with epsm.plan(pattern) as p:
        assert p.index_values() == want


def test_index_values_union_and_limit(epsm):
    pats = [b"ab", b"bc", b"cd" * 4, b"qrstuvwxyz"]      # the last one does not qualify
    assert epsm.index_values(pats) == b"abcd"
    many = [bytes([v, (v + 1) % 256]) for v in range(0, 256, 2)]
    assert len(epsm.index_values(many)) == 256
    assert epsm.index_values(many, limit=100) == b""     # a batch needing more than limit
    assert epsm.index_values([]) == b""


def test_index_entry_points_reject_bad_arguments(epsm):
    from paper_1209_6449_b200 import _lib
    lib = _lib._lib
    assert lib.epsm_eqidx_create(None) == epsm.EPSM_EINVAL
    h = ctypes.c_void_p()
    assert lib.epsm_eqidx_create(ctypes.byref(h)) == epsm.EPSM_OK
    try:
        vals = ctypes.create_string_buffer(b"ab", 2)
        # nv out of range, NULL values: rejected before any device work
        assert lib.epsm_eqidx_build_async(h, None, 0, vals, 0, None) == epsm.EPSM_EINVAL
        assert lib.epsm_eqidx_build_async(h, None, 0, None, 2, None) == epsm.EPSM_EINVAL
        assert lib.epsm_eqidx_build_async(h, None, 0, vals, 257, None) == epsm.EPSM_EINVAL
        # a misaligned text pointer
        assert lib.epsm_eqidx_build_async(h, 0x1001, 64, vals, 2, None) == epsm.EPSM_EALIGN
        dup = ctypes.create_string_buffer(b"aa", 2)
        assert lib.epsm_eqidx_build_async(h, 0x1000, 64, dup, 2, None) == epsm.EPSM_EINVAL
        assert lib.epsm_eqidx_values(h, None) == 0           # nothing built yet
    finally:
        lib.epsm_eqidx_free(h)
    lib.epsm_eqidx_free(None)                                # NULL-safe
