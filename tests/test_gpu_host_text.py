"""GPU parity of the end-to-end host call epsm_search_text_host: one HOST text, several groups
of patterns (the paper's protocol per text), positions copied into HOST
arrays.  Every search must return its own Occ(p, t) as the oracle computes it;
the dense searches run over an index the call builds itself, the copies of one group overlap
the next group's search, and capacities below occ keep the smallest positions."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

TILE = 32768


@pytest.fixture(scope="module")
def epsm():
    import paper_1209_6449_b200 as e
    return e


@pytest.mark.parametrize("sigma", [2, 4, 64])
def test_text_host_groups(epsm, sigma):
    torch.cuda.set_device(0)
    rng = np.random.default_rng(300 + sigma)
    n = 11 * TILE + 321
    t = rng.integers(0, sigma, size=n, dtype=np.uint8)
    groups, pats_all = [], []
    for m in (2, 3, 8, 17, 32):
        pats = [t[s:s + m].tobytes() for s in rng.integers(0, n - m + 1, size=12)]
        pats.append(bytes([255]) * m)                       # absent (sigma < 256)
        groups.append(epsm.group(pats))
        pats_all += pats
    wants = [oracle.search(p, t) for p in pats_all]
    if sigma == 2:
        assert any(len(g.index_values()) > 0 for g in groups)
    host_text = torch.from_numpy(t).pin_memory()
    outs = [torch.full((w.size + 3,), -5, dtype=torch.int64).pin_memory() for w in wants]
    caps = [w.size + 3 for w in wants]
    caps[0] = max(0, wants[0].size // 2)                   # a capacity below occ
    for rep in range(2):                                   # buffers reused by the second call
        occ = epsm.search_text_host(groups, host_text, outs, caps=caps)
        for j, w in enumerate(wants):
            assert int(occ[j]) == w.size, (rep, j)
            c = min(w.size, caps[j])
            assert np.array_equal(outs[j][:c].numpy().astype(np.uint64), w[:c]), (rep, j, len(pats_all[j]))
            if c < outs[j].numel() and caps[j] < w.size:
                assert int(outs[j][c]) == -5
    # counts only, pageable text
    occ = epsm.search_text_host(groups, t)
    assert [int(x) for x in occ] == [w.size for w in wants]
    for g in groups:
        g.close()


def test_text_host_edges(epsm):
    torch.cuda.set_device(0)
    g = epsm.group([b"ab", b"zz"])
    for text in (b"", b"a", b"ab", b"abab" * 5000 + b"a"):
        t = np.frombuffer(text, np.uint8).copy() if text else np.zeros(0, np.uint8)
        outs = [np.zeros(len(text) + 1, np.int64), np.zeros(len(text) + 1, np.int64)]
        occ = epsm.search_text_host([g], t, outs)
        for j, p in enumerate((b"ab", b"zz")):
            w = oracle.search(p, t)
            assert int(occ[j]) == w.size and np.array_equal(outs[j][:w.size].astype(np.uint64), w)
    g.close()
