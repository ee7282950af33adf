"""Thin ctypes binding of the C ABI in include/epsm.h (argument marshalling only).

Every step of the search runs in libepsm.so's sm_100a kernels; this module only
converts torch tensors / numpy arrays / CUDA streams into the pointers and sizes
the C calls take.  There is no CPU fallback: if libepsm.so is missing the import
fails, and on a machine without a GPU the calls raise EpsmError(EPSM_ECUDA).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libepsm.so")

EPSM_OK = 0
EPSM_EINVAL = -1
EPSM_EUNSUP = -2
EPSM_EALIGN = -3
EPSM_ECUDA = -4
EPSM_ENCCL = -5
EPSM_ENOMEM = -6
MAX_M = 32          # short patterns (packed / sampled filters in shared memory)
MAX_M_LONG = 4096   # long patterns (sampled filter, naive check against device memory)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: the CUDA extension was not built "
        "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)
_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p

_lib.epsm_plan.argtypes = [_vp, ctypes.c_uint32, ctypes.POINTER(_vp)]
_lib.epsm_plan.restype = ctypes.c_int
_lib.epsm_plan_free.argtypes = [_vp]
_lib.epsm_plan_free.restype = None
_lib.epsm_plan_m.argtypes = [_vp]
_lib.epsm_plan_m.restype = ctypes.c_uint32
_lib.epsm_count.argtypes = [_vp, _vp, _u64, _vp]
_lib.epsm_count.restype = _i64
_lib.epsm_count_async.argtypes = [_vp, _vp, _u64, _vp, _vp]
_lib.epsm_count_async.restype = ctypes.c_int
_lib.epsm_search.argtypes = [_vp, _vp, _u64, _vp, _u64, _vp]
_lib.epsm_search.restype = _i64
_lib.epsm_search_async.argtypes = [_vp, _vp, _u64, _vp, _u64, _vp, _vp]
_lib.epsm_search_async.restype = ctypes.c_int
_lib.epsm_search_batch_async.argtypes = [_vp, ctypes.c_uint32, _vp, _u64, _vp, _vp, _vp, _vp]
_lib.epsm_search_batch_async.restype = ctypes.c_int
_lib.epsm_count_batch_async.argtypes = [_vp, ctypes.c_uint32, _vp, _u64, _vp, _vp]
_lib.epsm_count_batch_async.restype = ctypes.c_int
_lib.epsm_search_range_batch_async.argtypes = [_vp, ctypes.c_uint32, _vp, _u64, _u64, _u64, _u64, _vp, _vp, _vp, _vp]
_lib.epsm_search_range_batch_async.restype = ctypes.c_int
_lib.epsm_search_host.argtypes = [_vp, _vp, _u64, _vp, _u64, _vp]
_lib.epsm_search_host.restype = _i64
_lib.epsm_search_sharded.argtypes = [_vp, _vp, _u64, _u64, _u64, _u64, _vp, _u64, _vp, _vp]
_lib.epsm_search_sharded.restype = _i64
_lib.epsm_search_range_async.argtypes = [_vp, _vp, _u64, _u64, _u64, _u64, _vp, _u64, _vp, _vp]
_lib.epsm_search_range_async.restype = ctypes.c_int
_lib.epsm_strerror.argtypes = [_i64]
_lib.epsm_strerror.restype = ctypes.c_char_p
_lib.epsm_last_error.argtypes = []
_lib.epsm_last_error.restype = ctypes.c_char_p
_lib.epsm_launch_count.argtypes = []
_lib.epsm_launch_count.restype = _u64
_lib.epsm_ktimer_enable.argtypes = [ctypes.c_int]
_lib.epsm_ktimer_enable.restype = ctypes.c_int
_lib.epsm_ktimer_read.argtypes = [ctypes.POINTER(_u64), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
_lib.epsm_ktimer_read.restype = ctypes.c_int
_lib.epsm_version.argtypes = []
_lib.epsm_version.restype = ctypes.c_int
_lib.epsm_debug_trace.argtypes = [_vp, _u64]
_lib.epsm_debug_trace.restype = _i64
_lib.epsm_eqidx_create.argtypes = [ctypes.POINTER(_vp)]
_lib.epsm_eqidx_create.restype = ctypes.c_int
_lib.epsm_eqidx_free.argtypes = [_vp]
_lib.epsm_eqidx_free.restype = None
_lib.epsm_eqidx_build_async.argtypes = [_vp, _vp, _u64, _vp, ctypes.c_uint32, _vp]
_lib.epsm_eqidx_build_async.restype = ctypes.c_int
_lib.epsm_eqidx_values.argtypes = [_vp, _vp]
_lib.epsm_eqidx_values.restype = ctypes.c_int
_lib.epsm_plan_index_values.argtypes = [_vp, _vp]
_lib.epsm_plan_index_values.restype = ctypes.c_int
_lib.epsm_search_range_batch_index_async.argtypes = [_vp, ctypes.c_uint32, _vp, _vp, _u64, _u64, _u64, _u64, _vp,
                                                     _vp, _vp, _vp]
_lib.epsm_search_range_batch_index_async.restype = ctypes.c_int
_lib.epsm_count_batch_index_async.argtypes = [_vp, ctypes.c_uint32, _vp, _vp, _u64, _vp, _vp]
_lib.epsm_count_batch_index_async.restype = ctypes.c_int
_lib.epsm_search_batch_index_async.argtypes = [_vp, ctypes.c_uint32, _vp, _vp, _u64, _vp, _vp, _vp, _vp]
_lib.epsm_search_batch_index_async.restype = ctypes.c_int

_lib.epsm_group_create.argtypes = [_vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(_vp)]
_lib.epsm_group_create.restype = ctypes.c_int
_lib.epsm_group_free.argtypes = [_vp]
_lib.epsm_group_free.restype = None
_lib.epsm_group_set_geometry.argtypes = [_vp, ctypes.c_uint32, ctypes.c_uint32]
_lib.epsm_group_set_geometry.restype = ctypes.c_int
_lib.epsm_group_info.argtypes = [_vp, _vp, ctypes.c_uint32]
_lib.epsm_group_info.restype = ctypes.c_int
_lib.epsm_group_search_async.argtypes = [_vp, _vp, _u64, _vp, _vp, _vp, _vp]
_lib.epsm_group_search_async.restype = ctypes.c_int
_lib.epsm_group_count_async.argtypes = [_vp, _vp, _u64, _vp, _vp]
_lib.epsm_group_count_async.restype = ctypes.c_int
_lib.epsm_group_search_range_async.argtypes = [_vp, _vp, _u64, _u64, _u64, _u64, _vp, _vp, _vp, _vp]
_lib.epsm_group_search_range_async.restype = ctypes.c_int
_lib.epsm_allgatherv_async.argtypes = [ctypes.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.epsm_allgatherv_async.restype = ctypes.c_int
_lib.epsm_group_dense_searches.argtypes = [_vp, _vp]
_lib.epsm_group_dense_searches.restype = ctypes.c_int
_lib.epsm_group_index_values.argtypes = [_vp, _vp]
_lib.epsm_group_index_values.restype = ctypes.c_int
_lib.epsm_search_text_host.argtypes = [_vp, ctypes.c_uint32, _vp, _u64, _vp, _vp, _vp, _vp]
_lib.epsm_search_text_host.restype = ctypes.c_int
_lib.epsm_group_set_dense.argtypes = [_vp, ctypes.c_uint32]
_lib.epsm_group_set_dense.restype = ctypes.c_int
_lib.epsm_group_search_index_async.argtypes = [_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp]
_lib.epsm_group_search_index_async.restype = ctypes.c_int
_lib.epsm_group_count_index_async.argtypes = [_vp, _vp, _vp, _u64, _vp, _vp]
_lib.epsm_group_count_index_async.restype = ctypes.c_int
_lib.epsm_group_search_range_index_async.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _u64, _vp, _vp, _vp, _vp]
_lib.epsm_group_search_range_index_async.restype = ctypes.c_int

EXPORTED_SYMBOLS = (
    "epsm_plan", "epsm_plan_free", "epsm_plan_m", "epsm_count", "epsm_count_async",
    "epsm_search", "epsm_search_async", "epsm_search_batch_async", "epsm_search_range_batch_async", "epsm_count_batch_async",
    "epsm_search_host", "epsm_search_sharded",
    "epsm_search_range_async", "epsm_strerror", "epsm_last_error", "epsm_launch_count",
    "epsm_ktimer_enable", "epsm_ktimer_read",
    "epsm_version", "epsm_debug_trace",
    "epsm_eqidx_create", "epsm_eqidx_free", "epsm_eqidx_build_async", "epsm_eqidx_values",
    "epsm_search_batch_index_async", "epsm_count_batch_index_async", "epsm_plan_index_values",
    "epsm_search_range_batch_index_async",
    "epsm_group_create", "epsm_group_free", "epsm_group_info", "epsm_group_set_geometry", "epsm_group_search_async",
    "epsm_group_count_async", "epsm_group_search_range_async", "epsm_group_set_dense",
    "epsm_group_search_index_async", "epsm_group_count_index_async", "epsm_group_search_range_index_async",
    "epsm_group_index_values", "epsm_search_text_host", "epsm_allgatherv_async", "epsm_group_dense_searches",
)
MAX_PLANES = 256
INDEX_MAX_D = 8


class EpsmError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = int(code)
        detail = _lib.epsm_last_error().decode(errors="replace")
        super().__init__(f"{where}: {strerror(code)}" + (f" ({detail})" if detail else ""))


def strerror(code: int) -> str:
    return _lib.epsm_strerror(int(code)).decode()


def launch_count() -> int:
    """Kernels libepsm.so has launched in this process so far."""
    return int(_lib.epsm_launch_count())


def ktimer_enable(on: bool) -> None:
    """Bracket every fan-out kernel launch with CUDA events (benchmark instrumentation)."""
    _check(_lib.epsm_ktimer_enable(1 if on else 0), "epsm_ktimer_enable")


def ktimer_read() -> tuple:
    """(launches, total ms, algorithmic bytes) of the fan-out launches recorded since the last read."""
    n, ms, b = _u64(0), ctypes.c_double(0.0), ctypes.c_double(0.0)
    _check(_lib.epsm_ktimer_read(ctypes.byref(n), ctypes.byref(ms), ctypes.byref(b)), "epsm_ktimer_read")
    return int(n.value), float(ms.value), float(b.value)


def version() -> int:
    return int(_lib.epsm_version())


def debug_trace() -> np.ndarray:
    """Per-launch, per-CTA timeline (EPSM_TRACE=<slots> runs only): uint64 [slots, 1024, 8]."""
    buf = np.zeros(1 << 22, dtype=np.uint64)
    k = _check(int(_lib.epsm_debug_trace(buf.ctypes.data, buf.size)), "epsm_debug_trace")
    return buf[:k].reshape(-1, 1024, 8)


def _check(rc: int, where: str) -> int:
    if rc < 0:
        raise EpsmError(rc, where)
    return rc


def _pattern_bytes(pattern) -> bytes:
    if isinstance(pattern, (bytes, bytearray, memoryview)):
        return bytes(pattern)
    if isinstance(pattern, str):
        return pattern.encode()
    if isinstance(pattern, torch.Tensor):
        return pattern.detach().cpu().contiguous().numpy().astype(np.uint8).tobytes()
    return np.asarray(pattern, dtype=np.uint8).tobytes()


class Plan:
    """epsm_plan(): the preprocessed pattern plus workspace."""

    def __init__(self, pattern):
        self.pattern = _pattern_bytes(pattern)
        h = _vp()
        buf = ctypes.create_string_buffer(self.pattern, max(len(self.pattern), 1))
        _check(_lib.epsm_plan(buf if self.pattern else None, len(self.pattern), ctypes.byref(h)), "epsm_plan")
        self._h = h

    @property
    def m(self) -> int:
        return len(self.pattern)

    def index_values(self) -> bytes:
        """epsm_plan_index_values: the bytes this search reads from an index (b"" if it never
        runs over one)."""
        buf = ctypes.create_string_buffer(8)
        d = _lib.epsm_plan_index_values(self.handle, buf)
        return buf.raw[:d]

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("plan is closed")
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None:
            _lib.epsm_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def plan(pattern) -> Plan:
    return Plan(pattern)


def _as_plan(p) -> Plan:
    return p if isinstance(p, Plan) else Plan(p)


def _stream_handle(stream, device) -> int:
    if stream is None:
        stream = torch.cuda.current_stream(device)
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _check_text(text: torch.Tensor):
    if not isinstance(text, torch.Tensor) or text.dtype != torch.uint8 or not text.is_cuda:
        raise TypeError("text must be a CUDA torch.uint8 tensor")
    if not text.is_contiguous():
        raise ValueError("text must be contiguous")


def _check_out(out: torch.Tensor | None, name: str):
    if out is None:
        return
    if not isinstance(out, torch.Tensor) or out.dtype not in (torch.int64, torch.uint64) or not out.is_cuda:
        raise TypeError(f"{name} must be a CUDA int64/uint64 tensor")
    if not out.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def count(p, text: torch.Tensor, stream=None) -> int:
    """|Occ(p, text)| for a CUDA uint8 text (synchronises the stream)."""
    pl = _as_plan(p)
    _check_text(text)
    return _check(_lib.epsm_count(pl.handle, text.data_ptr(), text.numel(),
                                  _stream_handle(stream, text.device)), "epsm_count")


def count_async(p: Plan, text: torch.Tensor, occ_out: torch.Tensor, stream=None) -> None:
    _check_text(text)
    _check_out(occ_out, "occ_out")
    _check(_lib.epsm_count_async(p.handle, text.data_ptr(), text.numel(), occ_out.data_ptr(),
                                 _stream_handle(stream, text.device)), "epsm_count_async")


def search(p, text: torch.Tensor, out: torch.Tensor | None = None, cap: int | None = None, stream=None):
    """Occurrences of the plan's pattern in ``text``.

    Returns ``(positions, occ)``: ``positions`` is the int64 CUDA tensor view
    ``out[:min(occ, cap)]`` (ascending), ``occ`` the full count.  Without ``out``
    a buffer is allocated (and grown once if it was too small)."""
    pl = _as_plan(p)
    _check_text(text)
    n = text.numel()
    strm = _stream_handle(stream, text.device)
    auto = out is None
    if auto:
        nst = max(0, n - pl.m + 1)
        size = min(nst, int(cap)) if cap is not None else min(nst, 1 << 16)
        out = torch.empty(size, dtype=torch.int64, device=text.device)
    _check_out(out, "out")
    c = out.numel() if cap is None else min(int(cap), out.numel())
    occ = _check(_lib.epsm_search(pl.handle, text.data_ptr(), n, out.data_ptr() if c else None, c, strm),
                 "epsm_search")
    if auto and cap is None and occ > c:
        out = torch.empty(occ, dtype=torch.int64, device=text.device)
        c = occ
        occ = _check(_lib.epsm_search(pl.handle, text.data_ptr(), n, out.data_ptr(), c, strm), "epsm_search")
    return out[: min(occ, c)], occ


def find_all(pattern, text: torch.Tensor) -> torch.Tensor:
    """All occurrence positions (int64 CUDA tensor, ascending)."""
    pos, _ = search(pattern, text)
    return pos


def search_async(p: Plan, text: torch.Tensor, out: torch.Tensor | None, occ_out: torch.Tensor,
                 cap: int | None = None, stream=None) -> None:
    """Enqueue a search; occ lands in occ_out[0] (device), positions in out."""
    _check_text(text)
    _check_out(out, "out")
    _check_out(occ_out, "occ_out")
    c = 0 if out is None else (out.numel() if cap is None else min(int(cap), out.numel()))
    _check(_lib.epsm_search_async(p.handle, text.data_ptr(), text.numel(),
                                  out.data_ptr() if (out is not None and c) else None, c,
                                  occ_out.data_ptr(), _stream_handle(stream, text.device)),
           "epsm_search_async")


def _batch_args(plans, text, occ_out, outs, caps):
    plans = [p if isinstance(p, Plan) else Plan(p) for p in plans]
    k = len(plans)
    _check_text(text)
    _check_out(occ_out, "occ_out")
    if occ_out.numel() < k:
        raise ValueError("occ_out needs one element per plan")
    hp = (ctypes.c_void_p * k)(*[p.handle.value for p in plans])
    pos_arr = caps_arr = None
    if outs is not None:
        ptrs, cs = [], []
        for j, o in enumerate(outs):
            _check_out(o, f"outs[{j}]")
            c = 0 if o is None else (o.numel() if caps is None else min(int(caps[j]), o.numel()))
            ptrs.append(o.data_ptr() if (o is not None and c) else None)
            cs.append(c)
        pos_arr = (ctypes.c_void_p * k)(*ptrs)
        caps_arr = (ctypes.c_uint64 * k)(*cs)
    return plans, k, hp, pos_arr, caps_arr


class EqIndex:
    """epsm_eqidx_*: the equality-mask planes of one text for a set of byte values
    (EPSMa's wscmp masks, computed once and shared by a batch)."""

    def __init__(self):
        h = _vp()
        _check(_lib.epsm_eqidx_create(ctypes.byref(h)), "epsm_eqidx_create")
        self._h = h
        self._text = None

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("index is closed")
        return self._h

    def build_async(self, text: torch.Tensor, values, stream=None) -> "EqIndex":
        """(Re)build the planes of `text` for the distinct byte values `values` on stream."""
        _check_text(text)
        vals = bytes(_pattern_bytes(values))
        buf = ctypes.create_string_buffer(vals, max(len(vals), 1))
        _check(_lib.epsm_eqidx_build_async(self.handle, text.data_ptr(), text.numel(), buf, len(vals),
                                           _stream_handle(stream, text.device)), "epsm_eqidx_build_async")
        self._text = text            # keep the text alive while the index refers to it
        return self

    @property
    def values(self) -> bytes:
        out = ctypes.create_string_buffer(MAX_PLANES)
        k = _lib.epsm_eqidx_values(self.handle, out)
        return out.raw[:k]

    def close(self):
        if getattr(self, "_h", None) is not None:
            _lib.epsm_eqidx_free(self._h)
            self._h = None
        self._text = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def eq_index(text: torch.Tensor, values, stream=None) -> EqIndex:
    """An EqIndex of `text` for `values` (built asynchronously on stream)."""
    return EqIndex().build_async(text, values, stream=stream)


def index_values(patterns, limit: int = MAX_PLANES) -> bytes:
    """Byte values an index needs for the searches among `patterns` that would run over one
    (epsm_plan_index_values), in first-seen order; empty if more than `limit` values."""
    seen = []
    buf = ctypes.create_string_buffer(INDEX_MAX_D)
    for p in patterns:
        pl = p if isinstance(p, Plan) else Plan(p)
        d = _lib.epsm_plan_index_values(pl.handle, buf)
        for v in buf.raw[:d]:
            if v not in seen:
                seen.append(v)
    return bytes(seen) if len(seen) <= limit else b""


def search_batch_async(plans, text: torch.Tensor, occ_out: torch.Tensor, outs=None, caps=None,
                       stream=None, index: EqIndex | None = None) -> None:
    """Enqueue len(plans) searches over one text (one persistent launch per run of equal m).

    occ_out: CUDA int64 tensor with >= len(plans) elements (occ of search j -> occ_out[j]).
    outs: None (count only) or a sequence of CUDA int64 tensors / None, one per plan;
    caps: optional sequence of capacities (default: each out's numel).
    index: an EqIndex built over this text: qualifying searches stream its planes.
    """
    if len(plans) == 0:
        return
    plans, k, hp, pos_arr, caps_arr = _batch_args(plans, text, occ_out, outs, caps)
    if index is not None:
        _check(_lib.epsm_search_batch_index_async(hp, k, index.handle, text.data_ptr(), text.numel(), pos_arr,
                                                  caps_arr, occ_out.data_ptr(),
                                                  _stream_handle(stream, text.device)),
               "epsm_search_batch_index_async")
        return
    _check(_lib.epsm_search_batch_async(hp, k, text.data_ptr(), text.numel(), pos_arr, caps_arr,
                                        occ_out.data_ptr(), _stream_handle(stream, text.device)),
           "epsm_search_batch_async")


def count_batch_async(plans, text: torch.Tensor, occ_out: torch.Tensor, stream=None,
                      index: "EqIndex | None" = None) -> None:
    """Enqueue len(plans) counts over one text (count kernel; occ of pattern j -> occ_out[j]);
    with an EqIndex of the text, qualifying searches count over its planes."""
    if len(plans) == 0:
        return
    plans, k, hp, _, _ = _batch_args(plans, text, occ_out, None, None)
    if index is not None:
        _check(_lib.epsm_count_batch_index_async(hp, k, index.handle, text.data_ptr(), text.numel(),
                                                 occ_out.data_ptr(), _stream_handle(stream, text.device)),
               "epsm_count_batch_index_async")
        return
    _check(_lib.epsm_count_batch_async(hp, k, text.data_ptr(), text.numel(), occ_out.data_ptr(),
                                       _stream_handle(stream, text.device)), "epsm_count_batch_async")


def search_range_batch_async(plans, shard: torch.Tensor, owned_len: int, base: int, n_total: int,
                             occ_out: torch.Tensor, outs=None, caps=None, stream=None,
                             index: "EqIndex | None" = None) -> None:
    """Local step of a sharded batch: starts s < owned_len of ``shard``, reported as s + base;
    n_total = the global text length (the shard must hold every owned window; with an EqIndex
    built over ``shard``, qualifying searches stream its planes)."""
    if len(plans) == 0:
        return
    plans, k, hp, pos_arr, caps_arr = _batch_args(plans, shard, occ_out, outs, caps)
    if index is not None:
        _check(_lib.epsm_search_range_batch_index_async(hp, k, index.handle, shard.data_ptr(), shard.numel(),
                                                        int(owned_len), int(base), int(n_total), pos_arr, caps_arr,
                                                        occ_out.data_ptr(), _stream_handle(stream, shard.device)),
               "epsm_search_range_batch_index_async")
        return
    _check(_lib.epsm_search_range_batch_async(hp, k, shard.data_ptr(), shard.numel(), int(owned_len), int(base),
                                              int(n_total), pos_arr, caps_arr, occ_out.data_ptr(),
                                              _stream_handle(stream, shard.device)),
           "epsm_search_range_batch_async")


def search_range_async(p: Plan, shard: torch.Tensor, owned_len: int, base: int, n_total: int,
                       out: torch.Tensor | None, occ_out: torch.Tensor, cap: int | None = None,
                       stream=None) -> None:
    """Local step of a sharded search: starts s < owned_len of ``shard``, reported as s + base
    (n_total = the global text length; the shard must hold every owned window)."""
    _check_text(shard)
    _check_out(out, "out")
    _check_out(occ_out, "occ_out")
    c = 0 if out is None else (out.numel() if cap is None else min(int(cap), out.numel()))
    _check(_lib.epsm_search_range_async(p.handle, shard.data_ptr(), shard.numel(), int(owned_len), int(base),
                                        int(n_total), out.data_ptr() if (out is not None and c) else None, c,
                                        occ_out.data_ptr(), _stream_handle(stream, shard.device)),
           "epsm_search_range_async")


def _host_ptr_len(a, dtype):
    if isinstance(a, torch.Tensor):
        if a.is_cuda or not a.is_contiguous():
            raise TypeError("host buffers must be contiguous CPU tensors or numpy arrays")
        return a.data_ptr(), a.numel()
    arr = np.asarray(a)
    if arr.dtype != dtype or not arr.flags["C_CONTIGUOUS"]:
        raise TypeError(f"host buffer must be a contiguous {dtype} array")
    return arr.ctypes.data, arr.size


def search_host(p, host_text, host_out=None, cap: int | None = None, stream=None) -> int:
    """epsm_search_host: host text in, host positions out (copies inside).  Returns occ."""
    pl = _as_plan(p)
    tp, n = _host_ptr_len(host_text, np.uint8)
    if host_out is None:
        op, c = None, 0
    else:
        op, c = _host_ptr_len(host_out, np.uint64)
        if cap is not None:
            c = min(c, int(cap))
    strm = _stream_handle(stream, None) if torch.cuda.is_available() else (stream or 0)
    return _check(_lib.epsm_search_host(pl.handle, tp, n, op if c else None, c, strm), "epsm_search_host")


def nccl_comm_ptr(group=None) -> int:
    """The ncclComm_t behind a torch.distributed NCCL process group."""
    import torch.distributed as dist
    g = group or dist.group.WORLD
    backend = g._get_backend(torch.device("cuda"))
    return int(backend._comm_ptr())


def search_sharded(p, shard: torch.Tensor, base: int, owned_len: int, n_total: int,
                   out: torch.Tensor | None = None, cap: int | None = None, group=None,
                   nccl_comm: int | None = None, stream=None) -> int:
    """epsm_search_sharded over a torch.distributed NCCL group (collective).

    Every rank ends with the first min(occ, cap) global positions in ``out``."""
    pl = _as_plan(p)
    _check_text(shard)
    _check_out(out, "out")
    comm = nccl_comm if nccl_comm is not None else nccl_comm_ptr(group)
    c = 0 if out is None else (out.numel() if cap is None else min(int(cap), out.numel()))
    return _check(_lib.epsm_search_sharded(pl.handle, shard.data_ptr(), int(base), int(owned_len),
                                           shard.numel(), int(n_total),
                                           out.data_ptr() if (out is not None and c) else None, c,
                                           comm, _stream_handle(stream, shard.device)),
                  "epsm_search_sharded")


class Group:
    """epsm_group_*: k patterns of one length searched in ONE pass over a text (the paper's
    protocol of many patterns per text); search j is patterns[j]."""

    def __init__(self, patterns):
        pats = [_pattern_bytes(p) for p in patterns]
        if not pats:
            raise ValueError("a group needs at least one pattern")
        m = len(pats[0])
        if any(len(p) != m for p in pats):
            raise ValueError("all patterns of a group have the same length")
        self.patterns = pats
        buf = ctypes.create_string_buffer(b"".join(pats), max(1, m * len(pats)))
        h = _vp()
        _check(_lib.epsm_group_create(buf, m, len(pats), ctypes.byref(h)), "epsm_group_create")
        self._h = h

    @property
    def m(self) -> int:
        return len(self.patterns[0])

    @property
    def k(self) -> int:
        return len(self.patterns)

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("group is closed")
        return self._h

    def info(self) -> dict:
        """{m, k, distinct, passes: [(q, SK), ...]} (epsm_group_info)."""
        out = (ctypes.c_uint32 * 64)()
        c = _check(_lib.epsm_group_info(self.handle, out, 64), "epsm_group_info")
        v = list(out[:min(c, 64)])
        return {"m": v[0], "k": v[1], "distinct": v[2], "dense": v[3],
                "passes": [(v[5 + 2 * i], v[6 + 2 * i]) for i in range(v[4])]}

    def set_geometry(self, q: int, sk: int) -> "Group":
        """Force sampled q-grams every SK bytes (tests / tuning; results never change)."""
        _check(_lib.epsm_group_set_geometry(self.handle, int(q), int(sk)), "epsm_group_set_geometry")
        return self

    def dense_searches(self) -> list:
        """flags[j] = True if search j is searched one by one (a dense pattern)."""
        out = (ctypes.c_uint8 * max(1, self.k))()
        _check(_lib.epsm_group_dense_searches(self.handle, out), "epsm_group_dense_searches")
        return [bool(x) for x in out[:self.k]]

    def index_values(self) -> bytes:
        """The byte values an equality-mask index needs for the dense searches."""
        out = (ctypes.c_uint8 * 256)()
        c = _lib.epsm_group_index_values(self.handle, out)
        return bytes(out[:c])

    def set_dense(self, log2_rate: int) -> "Group":
        """Re-split: patterns estimated at >= 2^-log2_rate occurrences per byte are searched one
        by one (0: none; tests / tuning, results never change)."""
        _check(_lib.epsm_group_set_dense(self.handle, int(log2_rate)), "epsm_group_set_dense")
        return self

    def _outs(self, outs, caps):
        k = self.k
        if outs is None:
            return None, None
        if len(outs) != k:
            raise ValueError("one output (or None) per search")
        ptrs, cs = [], []
        for j, o in enumerate(outs):
            _check_out(o, f"outs[{j}]")
            c = 0 if o is None else (o.numel() if caps is None else min(int(caps[j]), o.numel()))
            ptrs.append(o.data_ptr() if (o is not None and c) else None)
            cs.append(c)
        return (ctypes.c_void_p * k)(*ptrs), (ctypes.c_uint64 * k)(*cs)

    def search_async(self, text: torch.Tensor, occ_out: torch.Tensor, outs=None, caps=None, stream=None,
                     index: "EqIndex | None" = None):
        """Enqueue every search over ``text``: occ of search j -> occ_out[j], positions -> outs[j]
        (the dense patterns' searches over ``index`` where they qualify)."""
        _check_text(text)
        _check_out(occ_out, "occ_out")
        if occ_out.numel() < self.k:
            raise ValueError("occ_out needs one element per search")
        pa, ca = self._outs(outs, caps)
        st = _stream_handle(stream, text.device)
        if index is None:
            _check(_lib.epsm_group_search_async(self.handle, text.data_ptr(), text.numel(), pa, ca,
                                                occ_out.data_ptr(), st), "epsm_group_search_async")
        else:
            _check(_lib.epsm_group_search_index_async(self.handle, index.handle, text.data_ptr(), text.numel(), pa,
                                                      ca, occ_out.data_ptr(), st), "epsm_group_search_index_async")

    def count_async(self, text: torch.Tensor, occ_out: torch.Tensor, stream=None, index: "EqIndex | None" = None):
        _check_text(text)
        _check_out(occ_out, "occ_out")
        if occ_out.numel() < self.k:
            raise ValueError("occ_out needs one element per search")
        st = _stream_handle(stream, text.device)
        if index is None:
            _check(_lib.epsm_group_count_async(self.handle, text.data_ptr(), text.numel(), occ_out.data_ptr(), st),
                   "epsm_group_count_async")
        else:
            _check(_lib.epsm_group_count_index_async(self.handle, index.handle, text.data_ptr(), text.numel(),
                                                     occ_out.data_ptr(), st), "epsm_group_count_index_async")

    def search_range_async(self, shard: torch.Tensor, owned_len: int, base: int, n_total: int,
                           occ_out: torch.Tensor, outs=None, caps=None, stream=None, index: "EqIndex | None" = None):
        """Local step of a sharded group search (starts s < owned_len, reported as s + base)."""
        _check_text(shard)
        _check_out(occ_out, "occ_out")
        if occ_out.numel() < self.k:
            raise ValueError("occ_out needs one element per search")
        pa, ca = self._outs(outs, caps)
        _check(_lib.epsm_group_search_range_index_async(
            self.handle, None if index is None else index.handle, shard.data_ptr(), shard.numel(), int(owned_len),
            int(base), int(n_total), pa, ca, occ_out.data_ptr(), _stream_handle(stream, shard.device)),
            "epsm_group_search_range_index_async")

    def close(self):
        if getattr(self, "_h", None) is not None:
            _lib.epsm_group_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def group(patterns) -> Group:
    return Group(patterns)


def search_text_host(groups, host_text, host_outs=None, caps=None, stream=None) -> np.ndarray:
    """epsm_search_text_host: every search of every group over one HOST text (a pinned or
    pageable uint8 tensor / numpy array); search j's positions land in the host array
    host_outs[j] (searches numbered group by group).  Returns the occ of every search."""
    t, n = _host_ptr_len(host_text, np.uint8)
    ks = [g.k for g in groups]
    K = sum(ks)
    gp = (ctypes.c_void_p * len(groups))(*[g.handle for g in groups])
    pa = ca = None
    if host_outs is not None:
        if len(host_outs) != K:
            raise ValueError("one host output (or None) per search")
        ptrs, cs = [], []
        for j, o in enumerate(host_outs):
            if o is None:
                ptrs.append(None)
                cs.append(0)
                continue
            p, ln = _host_ptr_len(o, np.int64)
            ptrs.append(p)
            cs.append(ln if caps is None else min(int(caps[j]), ln))
        pa = (ctypes.c_void_p * K)(*ptrs)
        ca = (ctypes.c_uint64 * K)(*cs)
    occ = np.zeros(K, dtype=np.uint64)
    dev = torch.device("cuda", torch.cuda.current_device())
    _check(_lib.epsm_search_text_host(gp, len(groups), t, n, pa, ca, occ.ctypes.data, _stream_handle(stream, dev)),
           "epsm_search_text_host")
    return occ


def allgatherv_async(locals_, counts, outs, caps=None, nccl_comm=None, stream=None) -> None:
    """epsm_allgatherv_async: every rank's positions of search j (locals_[j], GLOBAL positions,
    device int64) into every rank's outs[j] at the prefix of counts ([world, k] host ints)."""
    k = len(locals_)
    cnt = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64).reshape(-1))
    if cnt.size % max(k, 1):
        raise ValueError("counts must be [world, k]")
    lp = (ctypes.c_void_p * k)(*[None if t is None else t.data_ptr() for t in locals_])
    op = (ctypes.c_void_p * k)(*[None if t is None else t.data_ptr() for t in outs])
    cp = None
    if caps is not None:
        cp = (ctypes.c_uint64 * k)(*[int(c) for c in caps])
    comm = nccl_comm if nccl_comm is not None else nccl_comm_ptr()
    dev = next((t.device for t in outs if t is not None), torch.device("cuda", torch.cuda.current_device()))
    _check(_lib.epsm_allgatherv_async(k, lp, cnt.ctypes.data, op, cp, ctypes.c_void_p(comm),
                                      _stream_handle(stream, dev)), "epsm_allgatherv_async")
