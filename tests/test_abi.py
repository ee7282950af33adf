"""The C ABI library loads and exports every symbol include/epsm.h declares, and
the host-side argument checks behave (no GPU needed: no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "epsm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(epsm_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("epsm_plan", "epsm_plan_free", "epsm_count", "epsm_search", "epsm_search_sharded",
              "epsm_search_async", "epsm_strerror"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_1209_6449_b200 as epsm
    lib = ctypes.CDLL(epsm.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(epsm.EXPORTED_SYMBOLS)


def test_no_oracle_or_torch_in_product_sources():
    """The product path never touches the oracle (and the kernels never see torch types)."""
    pkg = os.path.join(ROOT, "paper_1209_6449_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "epsm_oracle" not in txt, f
                if not f.endswith(".py"):
                    for bad in ("#include <torch", "#include <ATen", "at::Tensor", "c10::"):
                        assert bad not in txt, (f, bad)


def test_plan_argument_errors():
    import paper_1209_6449_b200 as epsm
    with pytest.raises(epsm.EpsmError) as e:
        epsm.plan(b"")
    assert e.value.code == epsm.EPSM_EINVAL
    with pytest.raises(epsm.EpsmError) as e:
        epsm.plan(b"x" * (epsm.MAX_M_LONG + 1))
    assert e.value.code == epsm.EPSM_EUNSUP
    for m in (1, 2, 4, 5, 16, 32, 33, 100, epsm.MAX_M_LONG):
        p = epsm.plan(b"q" * m)
        assert p.m == m
        p.close()
    assert "EINVAL" in epsm.strerror(-1)
    assert epsm.version() >= 100


def test_c_plan_direct():
    import paper_1209_6449_b200 as epsm
    lib = ctypes.CDLL(epsm.LIB_PATH)
    lib.epsm_plan.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_void_p)]
    lib.epsm_plan_m.argtypes = [ctypes.c_void_p]
    lib.epsm_plan_m.restype = ctypes.c_uint32
    lib.epsm_plan_free.argtypes = [ctypes.c_void_p]
    h = ctypes.c_void_p()
    assert lib.epsm_plan(ctypes.c_char_p(b"abc"), 3, ctypes.byref(h)) == 0
    assert lib.epsm_plan_m(h) == 3
    lib.epsm_plan_free(h)
    lib.epsm_plan_free(None)                      # NULL-safe
    assert lib.epsm_plan(None, 3, ctypes.byref(h)) == -1
    assert lib.epsm_plan(ctypes.c_char_p(b"abc"), 3, None) == -1
