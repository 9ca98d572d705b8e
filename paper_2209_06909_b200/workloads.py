"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's inputs are synthetic too; these are
the recipes of SURVEY.md section 8(d), all drawn from numpy's PCG64 via
``np.random.default_rng(np.random.SeedSequence(seed))`` like the reference
harness (harness.py:107).  Every generator takes ``n`` so that the parity
tests can run the same recipe at sizes the CPU oracle finishes in seconds.

Each generator returns ``keys`` (numpy array); the payload is always the
original index (int32), i.e. the reference's ``(key, index)`` records.
"""

from __future__ import annotations

import math
import os

import numpy as np

CONFIGS = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")

FULL_N = {"cfg1": 2**20, "cfg2": 2**24, "cfg3": 2**26, "cfg4": 2**26, "cfg5": 2**31}

DESCRIPTIONS = {
    "cfg1": "n=2^20 int32 uniform random permutation, k=4, min_run_len=24",
    "cfg2": "n=2^24 int32 random runs, lengths U[1,8192], half strictly descending, k=4",
    "cfg3": "n=2^26 int64 keys from 1024 distinct values, geometric runs (mean 4096), int32 index payload, k=4",
    "cfg4": "n=2^26 int32 skewed: one ascending run of n/2 then n/4 ascending pairs, k=4",
    "cfg5": "n=2^31 float32 uniform [-1e6,1e6], geometric ascending runs (mean 4096), k=4",
}


def _rng(seed):
    return np.random.default_rng(np.random.SeedSequence(seed))


def _truncated_lengths(draw, n):
    """Concatenate batches of positive lengths from ``draw(size)`` until they
    reach n; the last run is truncated so the lengths sum to exactly n."""
    out = []
    total = 0
    while total < n:
        batch = np.asarray(draw(max(16, n // 1024 + 16)), dtype=np.int64)
        csum = np.cumsum(batch) + total
        idx = np.searchsorted(csum, n, side="left")
        if idx < batch.shape[0]:
            part = batch[: idx + 1].copy()
            part[-1] = n - (csum[idx] - batch[idx])
            out.append(part)
            total = n
        else:
            out.append(batch)
            total = int(csum[-1])
    lengths = np.concatenate(out)
    assert int(lengths.sum()) == n and lengths.min() >= 1
    return lengths


def cfg1(n=FULL_N["cfg1"], seed=0):
    """Uniform random permutation of 0..n-1 (harness.generate
    "random-permutation", harness.py:108-109), int32."""
    return _rng(seed).permutation(n).astype(np.int32)


def cfg2(n=FULL_N["cfg2"], seed=0, max_len=None):
    """Random runs: lengths i.i.d. U[1, 2*sqrt(n)], values uniform int32
    sorted per run, each run reversed to strictly descending with p=0.5
    (equal neighbours fixed by a sequential decrement)."""
    if max_len is None:
        max_len = max(1, 2 * math.isqrt(n))
    rng = _rng(seed)
    lengths = _truncated_lengths(lambda size: rng.integers(1, max_len + 1, size=size), n)
    vals = rng.integers(-(2**31) + max_len, 2**31, size=n, dtype=np.int64)
    flips = rng.random(lengths.shape[0]) < 0.5
    out = np.empty(n, dtype=np.int64)
    pos = 0
    for length, flip in zip(lengths.tolist(), flips.tolist()):
        seg = np.sort(vals[pos : pos + length])
        if flip:
            seg = seg[::-1]
            # v[i] = min(v[i], v[i-1] - 1), sequentially (handles cascades)
            ramp = np.arange(length, dtype=np.int64)
            seg = np.minimum.accumulate(seg + ramp) - ramp
        out[pos : pos + length] = seg
        pos += length
    assert out.min() >= -(2**31) and out.max() < 2**31
    return out.astype(np.int32)


def cfg3(n=FULL_N["cfg3"], seed=0, distinct=1024, mean_len=4096):
    """Key-value stability stress: int64 keys from ``distinct`` values, laid
    out as ascending runs with geometric lengths of mean ``mean_len``."""
    rng = _rng(seed)
    palette = np.unique(rng.integers(-(2**62), 2**62, size=distinct * 2, dtype=np.int64))
    palette = rng.permutation(palette)[:distinct]
    keys = palette[rng.integers(0, palette.shape[0], size=n)]
    lengths = _truncated_lengths(lambda size: rng.geometric(1.0 / mean_len, size=size), n)
    pos = 0
    for length in lengths.tolist():
        keys[pos : pos + length].sort()
        pos += length
    return keys


def cfg4(n=FULL_N["cfg4"], seed=0):
    """Skewed profile: one ascending run of n/2 uniform int32, then n/4
    ascending pairs of uniform int32."""
    assert n % 4 == 0
    rng = _rng(seed)
    head = np.sort(rng.integers(-(2**31), 2**31, size=n // 2, dtype=np.int64))
    pairs = np.sort(rng.integers(-(2**31), 2**31, size=(n // 4, 2), dtype=np.int64), axis=1)
    return np.concatenate([head, pairs.reshape(-1)]).astype(np.int32)


CFG5_CHUNK = 2**24


def _cfg5_chunk(c, m, seed, mean_len):
    """Chunk c (m elements) of cfg5: its own PCG64 stream (SeedSequence([seed,
    c])), geometric run lengths truncated at the chunk end, and each run's
    values drawn directly in ascending order -- the order statistics of m
    uniforms are cumulative sums of exponential spacings, normalised by one
    extra spacing per run (no sort)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, c]))
    lengths = _truncated_lengths(lambda size: rng.geometric(1.0 / mean_len, size=size), m)
    r = lengths.shape[0]
    gaps = rng.standard_exponential(m + r)
    cs = np.cumsum(gaps)
    # run j occupies slots [s_j, s_j + L_j] of the spacings (L_j values + 1 gap)
    starts = np.concatenate(([0], np.cumsum(lengths + 1)[:-1]))
    base = np.where(starts > 0, cs[np.maximum(starts - 1, 0)], 0.0)
    total = cs[starts + lengths] - base
    keep = np.ones(m + r, dtype=bool)
    keep[starts + lengths] = False
    u = (cs[keep] - np.repeat(base, lengths)) / np.repeat(total, lengths)
    return (-1e6 + 2e6 * u).astype(np.float32)


def cfg5(n=FULL_N["cfg5"], seed=0, mean_len=4096, lo=0, hi=None, threads=None):
    """float32 uniform in [-1e6, 1e6] in ascending runs with geometric lengths
    of mean ``mean_len``.  Generated in independent chunks of 2^24 elements
    (runs end at chunk boundaries; adjacent runs may still fuse), so any
    chunk-aligned slice [lo, hi) -- a shard of the multi-GPU run -- is produced
    on its own, chunks in parallel on host threads."""
    from concurrent.futures import ThreadPoolExecutor

    hi = n if hi is None else hi
    C = min(CFG5_CHUNK, n)
    if lo % C or (hi % C and hi != n) or not 0 <= lo <= hi <= n:
        raise ValueError("cfg5 slices must be aligned to %d-element chunks" % C)
    out = np.empty(hi - lo, dtype=np.float32)
    chunks = list(range(lo // C, (hi + C - 1) // C))

    def one(c):
        a = c * C
        b = min(n, a + C)
        out[a - lo:b - lo] = _cfg5_chunk(c, b - a, seed, mean_len)

    workers = threads or min(len(chunks), os.cpu_count() or 1, 32)
    with ThreadPoolExecutor(max_workers=max(1, workers)) as ex:
        list(ex.map(one, chunks))
    return out


GENERATORS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


def generate(name, n=None, seed=0):
    gen = GENERATORS[name]
    return gen(FULL_N[name] if n is None else n, seed=seed)
