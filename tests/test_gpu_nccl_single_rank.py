"""The NCCL paths on real hardware with a one-rank communicator (the only multi-GPU code a
one-GPU box can execute): epsm_search_sharded (C ABI: dlopen'ed NCCL, counts all-gather,
grouped broadcasts of the positions) and the batched counts exchange over torch.distributed,
both against the oracle.  The multi-rank logic itself is covered over gloo on CPU
(tests/test_sharding.py)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        yield dist
    finally:
        dist.destroy_process_group()


def test_search_sharded_one_rank_matches_oracle(nccl_group):
    import paper_1209_6449_b200 as epsm
    from paper_1209_6449_b200 import sharding
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(61)
    n = 3 * 128 * 1024 + 777
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    comm = epsm.nccl_comm_ptr()
    for m in (2, 5, 8, 16, 32):
        p = t[999:999 + m].tobytes()
        want = oracle.search(p, t)
        base, owned, slen = sharding.shard_layout(n, 1, 0)
        out = torch.empty(want.size + 3, dtype=torch.int64, device=dev)
        occ = epsm.search_sharded(p, td[base:base + slen], base, owned, n, out=out, nccl_comm=comm)
        assert occ == want.size
        assert np.array_equal(out[:occ].cpu().numpy().astype(np.uint64), want)
        # truncated output: the cap smallest positions, full occ
        occ2 = epsm.search_sharded(p, td, 0, n, n, out=out, cap=max(1, want.size // 2), nccl_comm=comm)
        assert occ2 == want.size
        k = max(1, want.size // 2)
        assert np.array_equal(out[:k].cpu().numpy().astype(np.uint64), want[:k])


def test_batch_counts_exchange_over_nccl(nccl_group):
    import paper_1209_6449_b200 as epsm
    from paper_1209_6449_b200 import sharding
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(62)
    n = 2 * 128 * 1024 + 5
    t = rng.integers(0, 4, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    pats = [t[s:s + m].tobytes() for s, m in ((10, 2), (2000, 8), (70000, 16))]
    plans = [epsm.plan(p) for p in pats]
    occ_loc = torch.zeros(len(pats), dtype=torch.int64, device=dev)
    epsm.search_range_batch_async(plans, td, n, 0, n, occ_loc)
    occ, off = sharding.exchange_batch_counts(occ_loc)
    want = [oracle.search(p, t).size for p in pats]
    assert occ.cpu().tolist() == want and off.cpu().tolist() == [0] * len(pats)


def test_group_range_and_allgatherv_over_nccl(nccl_group):
    """The bench's N > 1 step on a one-rank communicator: group search over the shard (dense
    patterns over the shard's index), counts exchange, native positions all-gather
    (epsm_allgatherv_async) -- against the oracle."""
    import paper_1209_6449_b200 as epsm
    from paper_1209_6449_b200 import sharding
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(63)
    n = 5 * 128 * 1024 + 11
    t = rng.integers(0, 2, size=n, dtype=np.uint8)
    td = torch.from_numpy(t).to(dev)
    pats = [t[s:s + m].tobytes() for s, m in ((1, 2), (70, 2), (900, 8), (5000, 20), (9999, 32))]
    g = epsm.group(pats[:2])
    ix = epsm.eq_index(td, g.index_values()) if g.index_values() else None
    occ_loc = torch.zeros(2, dtype=torch.int64, device=dev)
    loc = [torch.empty(n, dtype=torch.int64, device=dev) for _ in range(2)]
    g.search_range_async(td, n, 0, n, occ_loc, outs=loc, index=ix)
    cm = sharding.exchange_count_matrix(occ_loc).cpu().numpy()
    outs = [torch.full((n,), -3, dtype=torch.int64, device=dev) for _ in range(2)]
    sharding.gather_batch_positions(loc, cm, outs, caps=[n, 5])
    torch.cuda.synchronize()
    for j in range(2):
        want = oracle.search(pats[j], t)
        c = want.size if j == 0 else 5
        assert int(cm[0, j]) == want.size
        assert np.array_equal(outs[j][:c].cpu().numpy().astype(np.uint64), want[:c])
        assert int(outs[j][c]) == -3
    g.close()
