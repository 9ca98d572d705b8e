"""Pin the CPU oracle (oracle/, a C++ restatement of the reference) against
golden vectors produced by the Python reference itself
(tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import oracle
from paper_2209_06909_b200 import workloads

NP_DTYPE = {"int32": np.int32, "int64": np.int64, "float32": np.float32}


def test_sorts_match_reference_bit_for_bit(golden_sorts):
    assert len(golden_sorts) > 300
    for case in golden_sorts:
        keys = np.array(case["keys"], dtype=NP_DTYPE[case["dtype"]])
        res = oracle.sort(keys, k=case["k"], variant=case["variant"], min_run_len=case["min_run_len"],
                          strict_merge_down=case["strict"])
        assert res.values.tolist() == case["perm"]
        want = dict(case["stats"])
        assert res.run_lengths == want.pop("run_lengths")
        assert res.natural_run_lengths == want.pop("natural_run_lengths")
        assert res.stats == want, (case["variant"], case["min_run_len"], case["strict"])
        assert [[list(b), l] for b, l in res.trace] == case["trace"]


def test_profiles_match_reference(golden_profiles):
    for case in golden_profiles:
        cost, trace, _ = oracle.merge_cost_for_profile(case["lengths"], case["k"], case["strict"])
        assert cost == case["cost"]
        assert [[list(b), l] for b, l in trace] == case["trace"]


def test_powers_match_reference(golden_powers):
    for k, n, b1, e1, b2, e2, p in golden_powers["powers"]:
        assert oracle.node_power(k, n, b1, e1, b2, e2) == p
    for k, n, cap in golden_powers["caps"]:
        assert oracle.run_stack_capacity(k, n) == cap
    assert golden_powers["node_power_2_4"] == oracle.node_power(2, 4, 0, 2, 2, 4) == 1


def test_reference_test_anchors():
    # tests/test_power.py:174-177 and :36-41 of the reference
    assert oracle.run_stack_capacity(4, 10**6) == 33
    assert oracle.run_stack_capacity(2, 16) == 5
    assert oracle.run_stack_capacity(4, 1) == 3
    with pytest.raises(ValueError):
        oracle.node_power(5, 4, 0, 2, 2, 4)
    with pytest.raises(ValueError):
        oracle.node_power(2, 4, 0, 2, 3, 4)
    # tests/test_policy.py:62-123
    cost, trace, _ = oracle.merge_cost_for_profile([2, 2, 4, 8], 4)
    assert cost == 20 and [(len(b) - 1, l) for b, l in trace] == [(2, 4), (3, 16)]
    cost, trace, _ = oracle.merge_cost_for_profile([2, 2, 4, 8], 2)
    assert cost == 28
    _, trace, _ = oracle.merge_cost_for_profile([4, 2, 2, 8], 2)
    assert trace == [((4, 6, 8), 4), ((0, 4, 8), 8), ((0, 8, 16), 16)]
    for stack_runs, arities in ((4, [4]), (5, [2, 4]), (6, [3, 4]), (7, [4, 4]), (9, [3, 4, 4])):
        prof = [2 ** (stack_runs - 1 - i) for i in range(stack_runs)]
        _, trace, _ = oracle.merge_cost_for_profile(prof, 4)
        assert [len(b) - 1 for b, _ in trace] == arities
    for stack_runs, arities in ((6, [4, 3]), (7, [4, 4]), (5, [4, 2])):
        prof = [2 ** (stack_runs - 1 - i) for i in range(stack_runs)]
        _, trace, _ = oracle.merge_cost_for_profile(prof, 4, strict_merge_down=True)
        assert [len(b) - 1 for b, _ in trace] == arities
    # sorted input: 0 merges, n-1 comparisons (tests/test_policy.py:29-38)
    res = oracle.sort(np.arange(1000, dtype=np.int32))
    assert res.stats["merge_cost"] == 0 and res.stats["comparisons"] == 999
    # the statskit golden (tests/test_statskit.py:24-36): 4M + 2n
    assert 4 * 678_233_797 + 2 * 10**8 == 2_912_935_188


def test_config_errors():
    with pytest.raises(ValueError):
        oracle.sort(np.arange(4, dtype=np.int32), k=3, variant="4way")
    with pytest.raises(ValueError):
        oracle.sort(np.arange(4, dtype=np.int32), k=2, variant="4way")
    with pytest.raises(ValueError):
        oracle.sort(np.arange(4, dtype=np.int32), min_run_len=0)


def sha(arr):
    return hashlib.sha256(np.asarray(arr, dtype=np.int64).tobytes()).hexdigest()


def test_cfg1_full_size_matches_reference(golden_cfg_full):
    g = golden_cfg_full["cfg1"]
    keys = workloads.generate("cfg1", n=g["n"], seed=g["seed"])
    assert hashlib.sha256(keys.tobytes()).hexdigest() == g["keys_sha256"]
    res = oracle.sort(keys)
    assert sha(res.values) == g["perm_sha256"]
    assert res.stats == g["stats"]
    assert sha(res.run_lengths) == g["run_lengths_sha256"]
    assert sha(res.natural_run_lengths) == g["natural_run_lengths_sha256"]
    flat = [x for b, l in res.trace for x in (len(b) - 1, *b, *([-1] * (5 - len(b))), l)]
    assert len(res.trace) == g["trace_len"] and sha(flat) == g["trace_sha256"]


def test_certificate_detects_errors():
    keys = np.array([3, 1, 2, 1], dtype=np.int32)
    perm = np.array([1, 3, 2, 0])
    assert oracle.stable_argsort_certificate(keys, keys[perm], perm) is None
    bad = np.array([3, 1, 2, 0])
    assert oracle.stable_argsort_certificate(keys, keys[bad], bad) is not None


def test_detect_runs_matches_reference_profiles(golden_sorts):
    # the read-only run chain (used at n = 2^31, where the full oracle cannot
    # run) against the reference's own run_lengths / natural_run_lengths
    for case in golden_sorts:
        keys = np.array(case["keys"], dtype=NP_DTYPE[case["dtype"]])
        if keys.size == 0:
            continue
        runs, nat = oracle.detect_runs(keys, case["min_run_len"])
        assert runs.tolist() == case["stats"]["run_lengths"]
        assert nat.tolist() == case["stats"]["natural_run_lengths"]


@pytest.mark.parametrize("name", workloads.CONFIGS)
def test_detect_runs_matches_full_oracle(name):
    keys = workloads.generate(name, n=1 << 18, seed=9)
    for mrl in (1, 24, 300):
        res = oracle.sort(keys, min_run_len=mrl, want_trace=False)
        runs, nat = oracle.detect_runs(keys, mrl)
        assert runs.tolist() == res.run_lengths and nat.tolist() == res.natural_run_lengths
