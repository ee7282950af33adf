"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds none of the method's arithmetic: it only generates texts and
extracts patterns.  Both the oracle side and the CUDA side read the bytes it
produces; neither side's results ever feed back into it.

Texts are counter-based: byte i depends only on (seed, i), so any shard
[start, start + count) can be generated on its own (needed for the multi-GPU
config, where each rank builds only its shard plus halo).  Byte i is drawn
from the 64-bit splitmix64 output z_i of the state key + (i+1) * GAMMA:

    uniform over an alphabet A:  A[(hi32(z_i) * |A|) >> 32]
    Zipf(s=1) over 27 symbols:   A_perm[searchsorted(CUM, hi32(z_i), 'right')]

The same recipe is implemented twice, in numpy (uint64) and in torch (int64
with masked logical shifts; runs on CPU or CUDA); tests/test_synth.py checks
that the two agree byte for byte.  The workloads mirror BASELINE.json configs
1-5, which stand in for the paper's Smart corpora (Sec. 4):
genome-like (ACGT), protein-like (20 amino-acid letters), natural-language-like
(Zipf over a-z + space) and random alphabets of size 2..256.  Patterns are
"randomly extracted from the text": starts are drawn
i.i.d. uniform over [0, n-m] with replacement (reading R12).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
M64 = (1 << 64) - 1

ACGT = b"ACGT"
PROTEIN = b"ACDEFGHIKLMNPQRSTVWY"
NL27 = b"abcdefghijklmnopqrstuvwxyz "

KiB = 1 << 10
MiB = 1 << 20
GiB = 1 << 30


def key_of(seed) -> int:
    """64-bit generator key from a seed word list (numpy SeedSequence)."""
    if isinstance(seed, int):
        seed = [seed]
    return int(np.random.SeedSequence(list(seed)).generate_state(1, dtype=np.uint64)[0])


def _s64(x: int) -> int:
    """Reinterpret an unsigned 64-bit constant as signed int64."""
    x &= M64
    return x - (1 << 64) if x >> 63 else x


def zipf_thresholds(k: int = 27, s: float = 1.0) -> np.ndarray:
    """Upper cumulative boundaries (k-1 of them) of Zipf(s) over ranks 1..k on
    the 32-bit integer line: rank index = searchsorted(th, u32, 'right')."""
    w = 1.0 / np.arange(1, k + 1, dtype=np.float64) ** s
    cum = np.cumsum(w / w.sum())[:-1]
    return np.floor(cum * 2.0 ** 32).astype(np.int64)


@dataclass(frozen=True)
class TextSpec:
    """A synthetic text: ``kind`` in {"uniform", "zipf", "unary"}."""
    kind: str
    alphabet: bytes
    seed: tuple = ()
    perm_seed: tuple = ()

    def sigma(self) -> int:
        return len(self.alphabet)

    def symbol_table(self) -> np.ndarray:
        a = np.frombuffer(self.alphabet, dtype=np.uint8).copy()
        if self.kind == "zipf":
            perm = np.random.default_rng(np.random.SeedSequence(list(self.perm_seed))).permutation(len(a))
            a = a[perm]
        return a


def uniform_spec(alphabet: bytes, seed) -> TextSpec:
    return TextSpec("uniform", bytes(alphabet), tuple(seed))


def raw_sigma_spec(sigma: int, seed) -> TextSpec:
    """Uniform over raw byte values 0..sigma-1 (BASELINE.json config 2)."""
    return TextSpec("uniform", bytes(range(sigma)), tuple(seed))


def zipf_spec(seed=(4,), perm_seed=(4, 0)) -> TextSpec:
    return TextSpec("zipf", NL27, tuple(seed), tuple(perm_seed))


def unary_spec(ch: bytes = b"a") -> TextSpec:
    return TextSpec("unary", bytes(ch))


# ---------------------------------------------------------------- numpy side

def _splitmix_np(key: int, start: int, count: int) -> np.ndarray:
    i = np.arange(start, start + count, dtype=np.uint64)
    z = np.uint64(key) + (i + np.uint64(1)) * np.uint64(GAMMA)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
    return z ^ (z >> np.uint64(31))


def text_np(spec: TextSpec, start: int, count: int) -> np.ndarray:
    """Bytes [start, start+count) of the text as a uint8 numpy array."""
    if count <= 0:
        return np.empty(0, dtype=np.uint8)
    table = spec.symbol_table()
    if spec.kind == "unary":
        return np.full(count, table[0], dtype=np.uint8)
    out = np.empty(count, dtype=np.uint8)
    key = key_of(spec.seed)
    step = 1 << 24
    with np.errstate(over="ignore"):
        for off in range(0, count, step):
            c = min(step, count - off)
            hi = (_splitmix_np(key, start + off, c) >> np.uint64(32)).astype(np.int64)
            if spec.kind == "uniform":
                idx = (hi * len(table)) >> 32
            else:
                idx = np.searchsorted(zipf_thresholds(len(table)), hi, side="right")
            out[off:off + c] = table[idx]
    return out


# ---------------------------------------------------------------- torch side

def _lshr(z, k: int):
    return (z >> k) & ((1 << (64 - k)) - 1)


def _splitmix_torch(key: int, start: int, count: int, device):
    import torch
    i = torch.arange(start + 1, start + count + 1, dtype=torch.int64, device=device)
    z = i * _s64(GAMMA) + _s64(key)
    z = (z ^ _lshr(z, 30)) * _s64(MIX1)
    z = (z ^ _lshr(z, 27)) * _s64(MIX2)
    return z ^ _lshr(z, 31)


def text_torch(spec: TextSpec, start: int, count: int, device="cpu", out=None, chunk: int = 1 << 26):
    """Bytes [start, start+count) as a torch.uint8 tensor on ``device`` (same
    bytes as text_np).  ``out`` may be a preallocated uint8 tensor of length
    >= count (only its first ``count`` bytes are written)."""
    import torch
    if out is None:
        out = torch.empty(count, dtype=torch.uint8, device=device)
    if count <= 0:
        return out
    table_np = spec.symbol_table()
    if spec.kind == "unary":
        out[:count].fill_(int(table_np[0]))
        return out
    table = torch.as_tensor(table_np, device=out.device)
    key = key_of(spec.seed)
    th = torch.as_tensor(zipf_thresholds(len(table_np)), device=out.device)
    for off in range(0, count, chunk):
        c = min(chunk, count - off)
        hi = _lshr(_splitmix_torch(key, start + off, c, out.device), 32)
        if spec.kind == "uniform":
            idx = (hi * len(table_np)) >> 32
        else:
            idx = torch.bucketize(hi, th, right=True)
        out[off:off + c] = table[idx]
        del hi, idx
    return out


# ---------------------------------------------------------------- patterns

def extract_starts(seed, n: int, m: int, count: int) -> np.ndarray:
    """Pattern starts i.i.d. uniform over [0, n-m] (PAPER.md:632 'randomly
    extracted'), seeded by a SeedSequence word list."""
    if n < m:
        raise ValueError("text shorter than pattern")
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(seed))))
    return rng.integers(0, n - m + 1, size=count, dtype=np.int64)


def extract_patterns_np(text: np.ndarray, seed, m: int, count: int):
    starts = extract_starts(seed, text.size, m, count)
    return [text[s:s + m].tobytes() for s in starts], starts


def extract_patterns_torch(text, seed, m: int, count: int):
    """Patterns copied out of a (device) torch uint8 text; returns (patterns, starts)."""
    import torch
    starts = extract_starts(seed, text.numel(), m, count)
    idx = torch.as_tensor(starts, device=text.device)[:, None] + torch.arange(m, device=text.device)[None, :]
    rows = text[idx].cpu().numpy()
    return [r.tobytes() for r in rows], starts


def extract_patterns_spec(spec: TextSpec, n: int, seed, m: int, count: int):
    """Patterns regenerated straight from the counter-based spec (no full text
    needed): pattern j = text[s_j : s_j + m]."""
    starts = extract_starts(seed, n, m, count)
    return [text_np(spec, int(s), m).tobytes() for s in starts], starts


# ---------------------------------------------------------------- configs

@dataclass
class Workload:
    """One (text, pattern set) group of a BASELINE.json config."""
    name: str
    spec: TextSpec
    n: int
    ms: tuple
    patterns_per_m: int
    start_seed: callable = field(repr=False, default=None)   # m -> seed words


def config_workloads(cfg: str):
    """The BASELINE.json configs as lists of Workloads (seeds per SURVEY 8(d))."""
    if cfg == "1":
        return [Workload("cfg1-acgt-1MiB", uniform_spec(ACGT, (1,)), 1 * MiB, (4,), 16,
                         lambda m: (1, 4, 1))]
    if cfg == "2":
        return [Workload(f"cfg2-sigma{s}-256MiB", raw_sigma_spec(s, (2, s)), 256 * MiB,
                         (2, 4, 8, 16, 32), 100, (lambda m, s=s: (2, s, m)))
                for s in (2, 4, 8, 16, 32, 64, 128, 256)]
    if cfg == "3":
        ms = (2, 3, 4, 6, 8, 12, 16, 20, 24, 28, 32)
        return [Workload("cfg3a-genome-1GiB", uniform_spec(ACGT, (3, 0)), 1 * GiB, ms, 100,
                         lambda m: (3, 0, m)),
                Workload("cfg3b-protein-1GiB", uniform_spec(PROTEIN, (3, 1)), 1 * GiB, ms, 100,
                         lambda m: (3, 1, m))]
    if cfg == "4":
        return [Workload("cfg4-zipf27-1GiB", zipf_spec(), 1 * GiB, (2, 4, 8, 16, 32), 100,
                         lambda m: (4, m))]
    if cfg == "5a":
        return [Workload("cfg5a-acgt-8GiB", uniform_spec(ACGT, (5,)), 8 * GiB, (8, 32), 100,
                         lambda m: (5, m))]
    if cfg == "5b":
        return [Workload("cfg5b-unary-1GiB", unary_spec(b"a"), 1 * GiB, (16,), 1, lambda m: (5, 1, m))]
    raise KeyError(cfg)
