"""Multi-rank host logic of the sharded search, world_size 2 (and 3) over gloo on
CPU.  The per-rank scan is the oracle here (no GPU); the layout, ownership,
halo and the counts/positions exchange are the production code."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1209_6449_b200 import sharding


def test_layout_partitions_starts():
    for n in (0, 1, 15, 16, 17, 1000, 1 << 20, (1 << 20) + 7):
        for world in (1, 2, 3, 4, 8):
            lay = sharding.all_layouts(n, world)
            assert lay[0][0] == 0
            covered = 0
            for r, (base, owned, slen) in enumerate(lay):
                assert base % 16 == 0
                assert base == covered
                covered += owned
                assert slen == min(n - base, owned + sharding.MAX_HALO)
            assert covered == n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    import torch
    import torch.distributed as dist
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for text, pattern, cap in cases:
            n = text.size
            base, owned, slen = sharding.shard_layout(n, world, rank)
            shard = torch.from_numpy(text[base:base + slen].copy())

            def local(sh, owned_len, b, n_total, p=pattern):
                # oracle over the shard, owned starts only, shifted to global
                pos = oracle.search(p, sh.numpy())
                pos = pos[pos < owned_len].astype(np.int64) + b
                return torch.from_numpy(pos), int(pos.size)

            pos, occ = sharding.search_sharded_torch(shard, base, owned, n, local, cap=cap)
            results.append((pos.numpy().copy(), occ))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_search_equals_unsharded(world):
    import oracle
    rng = np.random.default_rng(world)
    cases = []
    for n, sigma, m in [(5000, 2, 3), (40_000, 4, 8), (40_000, 4, 32), (33, 2, 2), (17, 256, 4)]:
        t = rng.integers(0, sigma, size=n, dtype=np.uint8)
        p = t[n // 3: n // 3 + m].copy()
        for r in range(1, world):   # occurrences straddling every cut
            b = sharding.shard_base(n, world, r)
            s = max(0, b - m // 2)
            if s + m <= n:
                t[s:s + m] = p
        cases.append((t, p.tobytes(), None))
        cases.append((t, p.tobytes(), 5))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for i, (t, p, cap) in enumerate(cases):
        want = oracle.search(p, t)
        for r in range(world):
            pos, occ = got[r][i]
            assert occ == want.size
            assert np.array_equal(pos.astype(np.uint64), want[:cap] if cap else want)


def _batch_worker(rank, world, port, text, patterns, q):
    import torch
    import torch.distributed as dist
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = text.size
        base, owned, slen = sharding.shard_layout(n, world, rank)
        shard = text[base:base + slen]
        local_pos, local_occ = [], []
        for p in patterns:
            pos = oracle.search(p, shard)
            pos = pos[pos < owned].astype(np.int64) + base
            local_pos.append(pos)
            local_occ.append(pos.size)
        occ, off = sharding.exchange_batch_counts(torch.tensor(local_occ, dtype=torch.int64))
        q.put((rank, occ.numpy().copy(), off.numpy().copy(), local_pos))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_batch_counts_exchange_gives_global_layout(world):
    """A sharded batch: every rank learns each search's global occ and its own offset, and the
    ranks' positions placed at those offsets are exactly Occ (oracle over the whole text)."""
    import oracle
    rng = np.random.default_rng(world + 40)
    n = 50_000
    text = rng.integers(0, 3, size=n, dtype=np.uint8)
    patterns = [text[s:s + m].tobytes() for s, m in ((7, 2), (1000, 5), (20_000, 9), (30_001, 17))]
    patterns.append(b"\x07\x07")                             # absent
    for r in range(1, world):                               # straddle every cut
        b = sharding.shard_base(n, world, r)
        text[b - 3:b - 3 + 9] = np.frombuffer(patterns[2], dtype=np.uint8)
    patterns = [text[s:s + m].tobytes() if i < 4 else p
                for i, (p, (s, m)) in enumerate(zip(patterns, ((7, 2), (1000, 5), (20_000, 9), (30_001, 17), (0, 2))))]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, text, patterns, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict((r, (o, f, lp)) for r, o, f, lp in (q.get(timeout=120) for _ in range(world)))
    for pr in procs:
        pr.join(timeout=60)
    for j, p in enumerate(patterns):
        want = oracle.search(p, text)
        out = np.full(want.size, -1, dtype=np.int64)
        for r in range(world):
            occ, off, lp = res[r]
            assert occ[j] == want.size
            out[off[j]: off[j] + lp[j].size] = lp[j]
        assert np.array_equal(out.astype(np.uint64), want)


def _gather_worker(rank, world, port, text, patterns, caps, q):
    import torch
    import torch.distributed as dist
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = text.size
        base, owned, slen = sharding.shard_layout(n, world, rank)
        shard = text[base:base + slen]
        local_outs, local_occ = [], []
        for p in patterns:
            pos = oracle.search(p, shard)
            pos = pos[pos < owned].astype(np.int64) + base
            local_outs.append(torch.from_numpy(pos.copy()))
            local_occ.append(pos.size)
        cm = sharding.exchange_count_matrix(torch.tensor(local_occ, dtype=torch.int64))
        tot = cm.sum(0)
        outs = [torch.full((int(t) + 2,), -9, dtype=torch.int64) for t in tot]
        sharding.gather_batch_positions(local_outs, cm.numpy(), outs, caps=caps)
        q.put((rank, [o.numpy().copy() for o in outs], tot.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_batch_positions_gather(world):
    """The N > 1 positions all-gather of a sharded batch (the bench's default multi-GPU exchange):
    every rank ends with every search's full Occ (oracle over the whole text), in order, the cap
    smallest when capped, nothing written past the cap."""
    import oracle
    rng = np.random.default_rng(world + 90)
    n = 60_000
    text = rng.integers(0, 2, size=n, dtype=np.uint8)
    patterns = [text[s:s + m].tobytes() for s, m in ((3, 2), (500, 6), (9000, 12), (40_000, 31))] + [b"\x05" * 3]
    for r in range(1, world):
        b = sharding.shard_base(n, world, r)
        text[b - 5:b - 5 + 12] = np.frombuffer(patterns[2], dtype=np.uint8)
    patterns[2] = bytes(text[9000:9012])
    caps = [10 ** 9, 7, 10 ** 9, 10 ** 9, 10 ** 9]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, text, patterns, caps, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict((r, (o, t)) for r, o, t in (q.get(timeout=120) for _ in range(world)))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for j, p in enumerate(patterns):
        want = oracle.search(p, text)
        c = min(want.size, caps[j])
        for r in range(world):
            outs, tot = res[r]
            assert tot[j] == want.size
            assert np.array_equal(outs[j][:c].astype(np.uint64), want[:c]), (r, j)
            assert (outs[j][c:] == -9).all()
