"""Full-size parity on the BASELINE configs, 1 GPU.

cfg2 (2^24 int32, k=4 and k=2), cfg3 (2^26 int64 key-value stress) and cfg4
(2^26 skewed profile) at their BASELINE sizes against the CPU oracle on the
same seeded input: the permutation and keys bit-exact, run_lengths and
natural_run_lengths, the merge tree in the reference's on_merge order
(policy.py:237-239), every SortStats field including comparisons and moves
(statskit.py:75-98) and scanned_elements_estimate (statskit.py:101-108).

cfg5 (2^31 float32) is beyond the full oracle (it would need the whole sort on
one host core and 32 GB of records), so it is checked by its parts: the O(n)
device certificate of the output (equivalent to bit-exactness),
the GPU run profile against the oracle's run chain on the same input
(runs.py:23-82, policy.py:241-248), and the executed merge tree, merge_cost
and max_stack_height against the oracle's merge_cost_for_profile on that
profile (policy.py:270-304).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import oracle  # noqa: E402
from paper_2209_06909_b200 import (  # noqa: E402
    SortConfig,
    merge_cost_for_profile,
    read_trace,
    scanned_elements_estimate,
    stable_argsort,
    workloads,
)
from paper_2209_06909_b200.certify import certify  # noqa: E402

STAT_FIELDS = ("comparisons", "merge_cost", "buffer_cost", "moves", "max_stack_height", "runs_detected", "merges2",
               "merges3", "merges4", "scan_reads", "scan_writes")


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available()
    return torch.device("cuda", 0)


@pytest.mark.parametrize("name,k", [("cfg2", 4), ("cfg2", 2), ("cfg3", 4), ("cfg4", 4)])
def test_full_size_vs_oracle(name, k, dev):
    n = workloads.FULL_N[name]
    keys_np = workloads.generate(name, seed=0)
    variant = "4way" if k == 4 else "2way"
    ref = oracle.sort(keys_np, k=k, variant=variant)
    keys = torch.from_numpy(keys_np).to(dev)
    out, perm, stats = stable_argsort(keys, SortConfig(k=k, variant=variant))
    assert np.array_equal(perm.cpu().numpy(), ref.values), "permutation"
    assert np.array_equal(out.cpu().numpy().view(np.uint8), ref.keys.view(np.uint8)), "keys"
    for f in STAT_FIELDS:
        assert getattr(stats, f) == ref.stats[f], f
    assert stats.run_lengths == ref.run_lengths
    assert stats.natural_run_lengths == ref.natural_run_lengths
    assert read_trace(device=dev) == ref.trace
    assert scanned_elements_estimate(stats, n) == 4 * ref.stats["merge_cost"] + 2 * n


def test_cfg5_full_size(dev):
    n = workloads.FULL_N["cfg5"]
    keys_np = workloads.generate("cfg5", seed=0)
    src = torch.from_numpy(keys_np).to(dev)
    keys = src.clone()
    _, perm, stats = stable_argsort(keys, SortConfig())
    certify(src, keys, perm)
    del src, keys, perm
    torch.cuda.empty_cache()
    # run profile against the oracle's run chain on the same input
    runs, nat = oracle.detect_runs(keys_np, 24)
    assert stats.runs_detected == runs.shape[0]
    assert np.array_equal(np.asarray(stats.run_lengths, dtype=np.int64), runs)
    assert np.array_equal(np.asarray(stats.natural_run_lengths, dtype=np.int64), nat)
    # the executed tree and its counters against the policy on that profile
    cost, trace, msh = oracle.merge_cost_for_profile(runs, 4)
    assert stats.merge_cost == cost
    assert stats.max_stack_height == msh
    assert read_trace(device=dev) == trace
    widths = [len(b) - 1 for b, _ in trace]
    assert (stats.merges2, stats.merges3, stats.merges4) == (widths.count(2), widths.count(3), widths.count(4))
    assert stats.scan_reads == n + 2 * cost
    assert stats.scan_writes == n + 2 * cost + 2 * stats.merges2 + 3 * stats.merges3 + 4 * stats.merges4
    assert scanned_elements_estimate(stats, n) == 4 * cost + 2 * n
    # and the device tree builder on the same profile
    assert merge_cost_for_profile(runs.tolist(), 4) == cost


def _adversarial(kind, n, seed=7):
    rng = np.random.default_rng(seed)
    if kind == "equal":
        return np.full(n, 5, dtype=np.int32)  # one run, every key tied
    if kind == "descending":
        return np.arange(n, 0, -1, dtype=np.int32)  # one strictly descending run (reversed)
    if kind == "zigzag":
        return np.tile(np.array([1, 0], dtype=np.int32), n // 2) + np.repeat(
            np.arange(n // 2, dtype=np.int32), 2)  # runs of two, every leaf an extended window
    if kind == "organ":
        h = np.arange(n // 2, dtype=np.int32)
        return np.concatenate([h, h[::-1]])  # one ascending run, then one descending
    if kind == "fewkeys_f64":
        return rng.integers(0, 3, size=n).astype(np.float64) * 0.5  # float64, three distinct keys
    if kind == "saw_i64":
        return (np.arange(n, dtype=np.int64) % 1000003) * (1 << 33)  # int64 ascending saw teeth
    raise ValueError(kind)


@pytest.mark.parametrize("kind,k", [("equal", 4), ("descending", 4), ("zigzag", 4), ("zigzag", 2), ("organ", 4),
                                    ("fewkeys_f64", 4), ("saw_i64", 2)])
def test_full_size_adversarial(kind, k, dev):
    """2^24-key adversarial inputs (ties everywhere, one reversed run, runs of
    two, two huge runs, float64 with three keys, int64 saw teeth) against the
    oracle: permutation, keys as bytes, run profile, trace and every counter."""
    n = 1 << 24
    keys_np = _adversarial(kind, n)
    variant = "4way" if k == 4 else "2way"
    ref = oracle.sort(keys_np, k=k, variant=variant)
    keys = torch.from_numpy(keys_np.copy()).to(dev)
    out, perm, stats = stable_argsort(keys, SortConfig(k=k, variant=variant))
    assert np.array_equal(perm.cpu().numpy(), ref.values), "permutation"
    assert np.array_equal(out.cpu().numpy().view(np.uint8), ref.keys.view(np.uint8)), "keys"
    for f in STAT_FIELDS:
        assert getattr(stats, f) == ref.stats[f], f
    assert stats.run_lengths == ref.run_lengths
    assert stats.natural_run_lengths == ref.natural_run_lengths
    assert read_trace(device=dev) == ref.trace
