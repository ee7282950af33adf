"""Data parallelism over the text (BASELINE.json north_star multi-GPU path).

The paper is single-threaded; sharding is this build's reading R11:

* the text of n bytes is cut into P contiguous pieces at 16-byte aligned
  boundaries base_r = round_down_16(r * n / P) (base_P = n);
* rank r OWNS the starts [base_r, base_{r+1}) and holds the bytes
  [base_r, min(n, base_{r+1} + halo)) with halo >= m - 1 (a fixed 31-byte halo
  serves every m <= 32), so every owned window lies inside its shard;
* every start belongs to exactly one rank, so the union of the per-rank
  occurrence sets is Occ(p, t) with no duplicates and no misses, and
  concatenating them in rank order keeps them sorted.

The exchange (counts, then positions) is the only collective.  This module
implements it with torch.distributed, so the same host logic runs over NCCL on
GPUs and over gloo on CPUs (tests/test_sharding.py).  The C ABI's
epsm_search_sharded does the same exchange natively with NCCL.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ALIGN = 16
MAX_HALO = 31   # m - 1 for the largest supported m (32)


def shard_base(n_total: int, world: int, rank: int) -> int:
    if rank >= world:
        return n_total
    return (rank * n_total // world) // ALIGN * ALIGN


def shard_layout(n_total: int, world: int, rank: int, halo: int = MAX_HALO):
    """(base, owned_len, shard_len) of ``rank``: owned starts [base, base+owned_len),
    bytes [base, base+shard_len)."""
    base = shard_base(n_total, world, rank)
    nxt = shard_base(n_total, world, rank + 1)
    owned = nxt - base
    shard_len = min(n_total - base, owned + halo)
    return base, owned, shard_len


def all_layouts(n_total: int, world: int, halo: int = MAX_HALO):
    return [shard_layout(n_total, world, r, halo) for r in range(world)]


def exchange_positions(local_pos: torch.Tensor, local_occ: int, group=None, cap: int | None = None):
    """All-gather per-rank counts, then the per-rank position lists.

    ``local_pos`` holds this rank's first min(local_occ, len) GLOBAL positions
    (ascending).  Returns (positions, occ) with positions = the first
    min(occ, cap) global positions in rank order, identical on every rank."""
    world = dist.get_world_size(group)
    dev = local_pos.device
    cnt = torch.tensor([int(local_occ)], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    occ = sum(counts)
    cap = occ if cap is None else min(int(cap), occ)
    keep, off = [], 0
    for c in counts:
        keep.append(max(0, min(c, cap - off)))
        off += c
    width = max(keep) if keep else 0
    if width == 0:
        return local_pos.new_empty(0), occ
    me = dist.get_rank(group)
    send = torch.zeros(width, dtype=torch.int64, device=dev)
    if keep[me]:
        send[: keep[me]] = local_pos[: keep[me]].to(torch.int64)
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    out = torch.cat([r[:k] for r, k in zip(recv, keep)])
    return out, occ


def exchange_count_matrix(local_occ: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather of a sharded batch's per-rank counts: returns [world, k] int64 (row q = rank
    q's local_occ) on local_occ's device.  One collective, no host synchronisation (NCCL)."""
    world = dist.get_world_size(group)
    k = local_occ.numel()
    dev = local_occ.device
    # gloo has no device all-gather: stage through the host (CPU tests, one-GPU emulation)
    via_host = dev.type == "cuda" and dist.get_backend(group) == "gloo"
    src = local_occ.reshape(-1).to(torch.int64)
    if via_host:
        src = src.cpu()
    allc = torch.empty(world * k, dtype=torch.int64, device=src.device)
    dist.all_gather_into_tensor(allc, src.contiguous(), group=group)
    if via_host:
        allc = allc.to(dev)
    return allc.view(world, k)


def gather_batch_positions(local_outs, counts, outs, caps=None, group=None) -> None:
    """The positions all-gather of a sharded batch of k searches (north_star: "allgathering the
    positions"): every rank's outs[j] receives the first min(occ_j, caps[j]) GLOBAL positions of
    search j in rank order -- rank q contributes counts[q][j] positions from its local_outs[j].
    ``counts`` is the [world, k] count matrix on the host (exchange_count_matrix(...).cpu()).
    NCCL: one native call (epsm_allgatherv_async: grouped ncclBroadcasts, one root per rank and
    search).  gloo (CPU tests, one-GPU emulation): a padded all-gather per search + placement."""
    import numpy as np
    cnt = np.asarray(counts, dtype=np.int64)
    world, k = cnt.shape
    if k == 0:
        return
    if dist.get_backend(group) == "nccl":
        from . import _lib
        _lib.allgatherv_async(local_outs, cnt, outs, caps=caps, nccl_comm=_lib.nccl_comm_ptr(group))
        return
    me = dist.get_rank(group)
    for j in range(k):
        width = int(cnt[:, j].max())
        if width == 0 or outs[j] is None:
            continue
        dev = outs[j].device
        send = torch.zeros(width, dtype=torch.int64)
        c_me = int(cnt[me, j])
        if c_me:
            send[:c_me] = local_outs[j][:c_me].to("cpu", torch.int64)
        recv = torch.empty(world * width, dtype=torch.int64)
        dist.all_gather_into_tensor(recv, send, group=group)
        recv = recv.view(world, width)
        cap = outs[j].numel() if caps is None else min(int(caps[j]), outs[j].numel())
        off = 0
        for q in range(world):
            c = min(int(cnt[q, j]), max(0, cap - off))
            if c:
                outs[j][off:off + c].copy_(recv[q, :c].to(dev))
            off += int(cnt[q, j])


def exchange_batch_counts(local_occ: torch.Tensor, group=None):
    """Counts exchange of a sharded batch of k searches (one all-gather of k int64 per rank).

    ``local_occ[j]`` = occurrences of search j among this rank's owned starts.  Returns
    (occ, offset): occ[j] = the global count, offset[j] = this rank's exclusive prefix (its
    positions of search j are the global positions [offset[j], offset[j] + local_occ[j]) of
    Occ in ascending order).  Stays on the device (no host synchronisation)."""
    rank = dist.get_rank(group)
    allc = exchange_count_matrix(local_occ, group)
    offset = allc.cumsum(0) - allc
    return allc.sum(0), offset[rank]


def search_sharded_torch(shard: torch.Tensor, base: int, owned_len: int, n_total: int, local_search,
                         group=None, cap: int | None = None):
    """Sharded search with the exchange done by torch.distributed.

    ``local_search(shard, owned_len, base) -> (global_positions, occ_local)`` is the
    per-rank scan (the CUDA path via ``local_search_cuda``; tests may inject the
    oracle to exercise this host logic on CPU)."""
    pos, occ_local = local_search(shard, owned_len, base, n_total)
    return exchange_positions(pos, occ_local, group=group, cap=cap)


def local_search_cuda(plan):
    """The per-rank scan through the C ABI (epsm_search_range_async)."""
    from . import _lib

    def run(shard: torch.Tensor, owned_len: int, base: int, n_total: int):
        occ_dev = torch.zeros(1, dtype=torch.int64, device=shard.device)
        nst = max(0, min(owned_len, shard.numel() - plan.m + 1))
        out = torch.empty(min(nst, 1 << 20), dtype=torch.int64, device=shard.device)
        _lib.search_range_async(plan, shard, owned_len, base, n_total, out, occ_dev)
        occ = int(occ_dev.item())
        if occ > out.numel():
            out = torch.empty(occ, dtype=torch.int64, device=shard.device)
            _lib.search_range_async(plan, shard, owned_len, base, n_total, out, occ_dev)
        return out[:occ], occ

    return run
