"""The paper's EPSM (SSE4.2) on the host CPU -- a second HOST BASELINE.

Not the oracle (``oracle/`` stays the brute force that pins parity) and not the product (the
CUDA library in ``paper_1209_6449_b200/``): it puts the paper's own x86 method (EPSMa / EPSMb /
EPSMc, Fig. 1) on the GPU box's host cores so that ``bench.py`` can time it
beside the oracle.  The arithmetic lives in ``epsm_sse.c``; this module marshals arguments
(ctypes, the GIL is released during a call) and runs one pattern per thread.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "epsm_sse.c")
_SO = os.path.join(_HERE, "libcpu_epsm.so")
_LOCK = threading.Lock()
_LIB = None
FLAGS = ["-O2", "-msse4.2", "-mpopcnt", "-std=gnu99"]


def build(force: bool = False) -> str:
    """gcc -O2 -msse4.2 -mpopcnt epsm_sse.c -> cpu_epsm/libcpu_epsm.so."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *FLAGS, "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def _lib():
    global _LIB
    with _LOCK:
        if _LIB is None:
            lib = ctypes.CDLL(build())
            lib.cpu_epsm_search.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                            ctypes.c_void_p, ctypes.c_uint64]
            lib.cpu_epsm_search.restype = ctypes.c_int64
            lib.cpu_epsm_variant.argtypes = [ctypes.c_uint64]
            lib.cpu_epsm_variant.restype = ctypes.c_int
            _LIB = lib
    return _LIB


def _u8(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    a = np.ascontiguousarray(x)
    if a.dtype != np.uint8:
        raise TypeError("uint8 text / pattern expected")
    return a.reshape(-1)


def variant(m: int) -> str:
    """The procedure EPSM's dispatch picks for length m: 'a', 'b' or 'c'."""
    return "abc"[_lib().cpu_epsm_variant(int(m))]


def search(pattern, text, cap: int | None = None) -> np.ndarray:
    """All occurrence positions (ascending uint64) of pattern in text."""
    p, t = _u8(pattern), _u8(text)
    if p.size == 0:
        raise ValueError("empty pattern")
    lib = _lib()
    if cap is None:
        occ = lib.cpu_epsm_search(p.ctypes.data, p.size, t.ctypes.data, t.size, None, 0)
        cap = occ
    out = np.empty(max(int(cap), 1), dtype=np.uint64)
    occ = lib.cpu_epsm_search(p.ctypes.data, p.size, t.ctypes.data, t.size, out.ctypes.data, int(cap))
    return out[:min(int(occ), int(cap))]


def count(pattern, text) -> int:
    p, t = _u8(pattern), _u8(text)
    if p.size == 0:
        raise ValueError("empty pattern")
    return int(_lib().cpu_epsm_search(p.ctypes.data, p.size, t.ctypes.data, t.size, None, 0))


def search_many(patterns, text, threads: int | None = None, positions: bool = True):
    """One pattern per thread (the GIL is released inside the C call)."""
    t = _u8(text)
    threads = threads or len(os.sched_getaffinity(0))
    f = (lambda p: search(p, t)) if positions else (lambda p: count(p, t))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(f, patterns))
