"""GPU parity fuzz: seeded random run structures, key types, variants and
min_run_len through the C ABI against the CPU oracle -- permutation, keys as
bytes, run profile, trace and every SortStats field (policy.py:201-262,
statskit.py:75-98).  PS_FUZZ_TRIALS sets the trial count (default 24)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import oracle  # noqa: E402
from paper_2209_06909_b200 import SortConfig, read_trace, stable_argsort  # noqa: E402
from paper_2209_06909_b200.policy import check  # noqa: E402

FIELDS = ("merge_cost", "max_stack_height", "runs_detected", "merges2", "merges3", "merges4", "buffer_cost",
          "scan_reads", "scan_writes", "moves", "comparisons")
VARIANTS = {"2way": 2, "2way-copy-smaller": 2, "2way-nosentinel": 2, "4way": 4, "4way-nosentinel": 4}
DTYPES = (np.int32, np.float32, np.int64, np.float64)


def make_input(rng, dtype):
    """Runs whose lengths mix the kernels' regimes: windows, tiny / mid nodes,
    chunks around the pipe units' capacities, a few long runs; ties and
    descending runs included."""
    target = int(rng.choice([3_000, 60_000, 400_000, 1_500_000, 3_000_000]))
    style = int(rng.integers(0, 5))
    parts, n = [], 0
    while n < target:
        if style == 0:
            ln = int(rng.integers(1, 64))
        elif style == 1:
            ln = int(rng.geometric(1 / 700.0))
        elif style == 2:
            ln = int(rng.choice([1076, 1077, 2152, 4305, 4320, 4576, 8640])) + int(rng.integers(-2, 3))
        elif style == 3:
            ln = int(rng.choice([5, 30, 300, 3000, 30000, 300000]))
        else:
            ln = int(rng.integers(1, 200_000)) if rng.random() < 0.1 else int(rng.integers(1, 40))
        ln = max(1, min(ln, target - n))
        span = int(rng.choice([3, 1000, 1 << 30]))
        v = np.sort(rng.integers(-span, span, ln))
        r = rng.random()
        if r < 0.3 and ln > 1:
            v = np.unique(v)[::-1]  # strictly descending
            ln = v.size
        parts.append(v)
        n += ln
    keys = np.concatenate(parts)
    if np.issubdtype(dtype, np.floating):
        keys = keys.astype(dtype) * dtype(0.5)
        if rng.random() < 0.5:  # signed zeros compare equal, their bytes differ
            z = rng.integers(0, keys.size, max(1, keys.size // 50))
            keys[z] = dtype(0.0)
            keys[z[::2]] = -dtype(0.0)
        return keys
    return keys.astype(dtype)


@pytest.mark.parametrize("seed", range(int(os.environ.get("PS_FUZZ_TRIALS", "24"))))
def test_fuzz_vs_oracle(seed):
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(90_000 + seed)
    dtype = DTYPES[seed % 4]
    variant = list(VARIANTS)[int(rng.integers(0, 5))]
    k = VARIANTS[variant]
    mrl = int(rng.choice([1, 2, 24, 24, 24, 40, 300]))
    strict = bool(rng.random() < 0.25)
    keys = make_input(rng, dtype)
    what = (seed, dtype.__name__, variant, mrl, strict, keys.size)
    ref = oracle.sort(keys, k=k, variant=variant, min_run_len=mrl, strict_merge_down=strict)
    out, perm, stats = stable_argsort(torch.from_numpy(keys).to(dev),
                                      SortConfig(k=k, variant=variant, min_run_len=mrl, strict_merge_down=strict))
    check(dev)
    torch.cuda.synchronize()
    assert np.array_equal(perm.cpu().numpy(), ref.values), what
    assert np.array_equal(out.cpu().numpy().view(np.uint8), ref.keys.view(np.uint8)), what
    for f in FIELDS:
        assert getattr(stats, f) == ref.stats[f], (f, what)
    assert stats.run_lengths == ref.run_lengths, what
    assert stats.natural_run_lengths == ref.natural_run_lengths, what
    assert read_trace(device=dev) == ref.trace, what
