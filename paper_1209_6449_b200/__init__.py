"""paper_1209_6449_b200 -- B200-native exact packed string matching (arXiv 1209.6449).

The hot path (every occurrence of a 1..32-byte pattern in a byte text, sorted
uint64 positions) runs in hand-written sm_100a kernels behind the C ABI in
include/epsm.h; this package is the thin Python binding over it.
"""
from ._lib import (  # noqa: F401
    EPSM_EALIGN, EPSM_ECUDA, EPSM_EINVAL, EPSM_ENCCL, EPSM_ENOMEM, EPSM_EUNSUP, EPSM_OK,
    EXPORTED_SYMBOLS, INDEX_MAX_D, Group, group, LIB_PATH, MAX_M, MAX_M_LONG, MAX_PLANES, EpsmError, EqIndex, Plan, count,
    eq_index, index_values, count_async, count_batch_async, find_all,
    debug_trace, ktimer_enable, ktimer_read, launch_count, nccl_comm_ptr, plan, search, search_async, search_batch_async, search_host, search_range_async,
    search_range_batch_async, search_text_host, allgatherv_async,
    search_sharded, strerror, version,
)
from . import sharding  # noqa: F401
