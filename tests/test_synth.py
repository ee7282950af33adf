"""The seeded generators: numpy and torch agree byte for byte, shards compose,
and the symbol distributions have the intended support."""
import numpy as np
import pytest
import torch

import synth


@pytest.mark.parametrize("spec", [
    synth.uniform_spec(synth.ACGT, (1,)),
    synth.raw_sigma_spec(2, (2, 2)),
    synth.raw_sigma_spec(256, (2, 256)),
    synth.uniform_spec(synth.PROTEIN, (3, 1)),
    synth.zipf_spec(),
    synth.unary_spec(),
])
def test_numpy_torch_agree_and_shards_compose(spec):
    n = 100_003
    a = synth.text_np(spec, 0, n)
    b = synth.text_torch(spec, 0, n, chunk=4096).numpy()
    assert np.array_equal(a, b)
    # any shard is the slice of the whole
    c = synth.text_np(spec, 777, 5000)
    assert np.array_equal(c, a[777:5777])
    d = synth.text_torch(spec, 99_000, 1003).numpy()
    assert np.array_equal(d, a[99_000:])
    assert set(np.unique(a).tolist()) <= set(spec.symbol_table().tolist())


def test_uniform_support_and_balance():
    a = synth.text_np(synth.raw_sigma_spec(4, (2, 4)), 0, 1 << 18)
    counts = np.bincount(a, minlength=256)
    assert counts[:4].min() > 0.24 * a.size and counts[4:].sum() == 0


def test_zipf_top_symbol_probability():
    a = synth.text_np(synth.zipf_spec(), 0, 1 << 18)
    p = np.bincount(a, minlength=256) / a.size
    top = p.max()
    assert abs(top - 1 / sum(1 / r for r in range(1, 28))) < 0.01   # 0.257
    assert (p > 0).sum() == 27


def test_pattern_extraction_is_seeded():
    spec = synth.uniform_spec(synth.ACGT, (1,))
    t = synth.text_np(spec, 0, 1 << 16)
    p1, s1 = synth.extract_patterns_np(t, (1, 4, 1), 4, 16)
    p2, s2 = synth.extract_patterns_spec(spec, t.size, (1, 4, 1), 4, 16)
    assert p1 == p2 and np.array_equal(s1, s2)
    assert all(t[s:s + 4].tobytes() == p for s, p in zip(s1, p1))
    pt, st = synth.extract_patterns_torch(torch.from_numpy(t), (1, 4, 1), 4, 16)
    assert pt == p1
