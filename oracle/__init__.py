"""CPU oracle for exact string matching -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product path (``paper_1209_6449_b200``) never imports it and shares no code
with it.

The arithmetic lives in ``epsm_oracle.c`` (plain C brute force of
Occ(p, t) = {s : 0 <= s <= n-m, t[s..s+m-1] = p}, Sec. 1);
this module only marshals arguments through ctypes.  ``build()`` compiles the
C file with gcc; ``_lib()`` compiles on first use if the .so is missing.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "epsm_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_LOCK = threading.Lock()
_LIB = None

EINVAL = -1


def build(force: bool = False) -> str:
    """Compile epsm_oracle.c into oracle/liboracle.so (portable -O2, no -march)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def _lib():
    global _LIB
    with _LOCK:
        if _LIB is None:
            lib = ctypes.CDLL(build())
            u8p = ctypes.c_void_p
            lib.oracle_search.argtypes = [u8p, ctypes.c_uint64, u8p, ctypes.c_uint64,
                                          ctypes.c_void_p, ctypes.c_uint64]
            lib.oracle_search.restype = ctypes.c_int64
            lib.oracle_count.argtypes = [u8p, ctypes.c_uint64, u8p, ctypes.c_uint64]
            lib.oracle_count.restype = ctypes.c_int64
            lib.oracle_verify.argtypes = [u8p, ctypes.c_uint64, u8p, ctypes.c_uint64,
                                          ctypes.c_uint64]
            lib.oracle_verify.restype = ctypes.c_int
            _LIB = lib
    return _LIB


def _as_u8(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    a = np.asarray(x)
    if a.dtype != np.uint8:
        raise TypeError(f"expected uint8 data, got {a.dtype}")
    return np.ascontiguousarray(a.reshape(-1))


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


def search(pattern, text, cap: int | None = None) -> np.ndarray:
    """Sorted uint64 positions of every occurrence of ``pattern`` in ``text``.

    With ``cap`` given, only the first ``cap`` positions are returned (the
    oracle still counts all of them; see ``search_capped``).
    """
    pos, _ = search_capped(pattern, text, cap)
    return pos


def search_capped(pattern, text, cap: int | None = None):
    """(positions[:min(occ, cap)], occ) -- mirrors the product's cap contract."""
    p = _as_u8(pattern)
    t = _as_u8(text)
    lib = _lib()
    if p.size == 0:
        raise ValueError("empty pattern (m = 0) is a usage error")
    if cap is None:
        occ = lib.oracle_count(_ptr(p), p.size, _ptr(t), t.size)
        cap = occ
    out = np.empty(max(int(cap), 0), dtype=np.uint64)
    occ = lib.oracle_search(_ptr(p), p.size, _ptr(t), t.size, _ptr(out), out.size)
    if occ < 0:
        raise ValueError(f"oracle_search error {occ}")
    return out[: min(occ, out.size)], int(occ)


def count(pattern, text) -> int:
    p = _as_u8(pattern)
    t = _as_u8(text)
    if p.size == 0:
        raise ValueError("empty pattern (m = 0) is a usage error")
    occ = _lib().oracle_count(_ptr(p), p.size, _ptr(t), t.size)
    if occ < 0:
        raise ValueError(f"oracle_count error {occ}")
    return int(occ)


def verify(pattern, text, s: int) -> bool:
    p = _as_u8(pattern)
    t = _as_u8(text)
    return bool(_lib().oracle_verify(_ptr(p), p.size, _ptr(t), t.size, int(s)))


def search_many(patterns, text, threads: int | None = None, count_only: bool = False):
    """Run the oracle for several patterns over one text on a thread pool.

    ctypes releases the GIL during the C call, so each worker thread runs one
    pattern's sequential scan on its own core.  Returns a list of position
    arrays (or of counts with ``count_only``) in the order of ``patterns``.
    """
    t = _as_u8(text)
    threads = threads or len(os.sched_getaffinity(0))
    fn = (lambda p: count(p, t)) if count_only else (lambda p: search(p, t))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, patterns))
