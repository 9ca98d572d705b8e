"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the CPU oracle on the BASELINE config recipes."""

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
    stable_sort_with,
    workloads,
)

NP_DTYPE = {"int32": np.int32, "int64": np.int64, "float32": np.float32}
POLICY_FIELDS = ("merge_cost", "max_stack_height", "runs_detected", "merges2", "merges3", "merges4")
COUNTER_FIELDS = ("buffer_cost", "scan_reads", "scan_writes")
VARIANTS = {"2way": 2, "2way-copy-smaller": 2, "2way-nosentinel": 2, "4way": 4, "4way-nosentinel": 4}



@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available()
    return torch.device("cuda", 0)


def gpu_sort(keys_np, dev, **cfg):
    from paper_2209_06909_b200.policy import check

    keys = torch.from_numpy(np.ascontiguousarray(keys_np)).to(dev)
    out, perm, stats = stable_argsort(keys, SortConfig(**cfg))
    check(dev)  # merge-phase device invariants
    torch.cuda.synchronize()
    return out.cpu().numpy(), perm.cpu().numpy(), stats


def test_golden_sorts(golden_sorts, dev):
    for case in golden_sorts:
        keys = np.array(case["keys"], dtype=NP_DTYPE[case["dtype"]])
        cfg = dict(k=case["k"], variant=case["variant"], min_run_len=case["min_run_len"],
                   strict_merge_down=case["strict"])
        if keys.size == 0:
            continue
        out, perm, stats = gpu_sort(keys, dev, count_comparisons=False, **cfg)
        assert perm.tolist() == case["perm"], cfg
        assert np.array_equal(out.view(np.uint8), keys[perm].view(np.uint8))
        want = case["stats"]
        for f in POLICY_FIELDS + COUNTER_FIELDS:
            assert getattr(stats, f) == want[f], (f, cfg)
        assert stats.comparisons is None and stats.moves is None
        # the default config counts, like the reference (statskit.py:49-72)
        _, perm2, cstats = gpu_sort(keys, dev, **cfg)
        assert perm2.tolist() == case["perm"], cfg
        assert cstats.moves == want["moves"], (cfg, keys.size)
        assert cstats.comparisons == want["comparisons"], (cfg, keys.size)
        assert stats.run_lengths == want["run_lengths"]
        assert stats.natural_run_lengths == want["natural_run_lengths"]
        assert [[list(b), l] for b, l in read_trace(device=dev)] == case["trace"], cfg


def test_golden_profiles(golden_profiles, dev):
    for case in golden_profiles:
        trace = []
        cost = merge_cost_for_profile(case["lengths"], case["k"], case["strict"], on_merge=trace.append)
        assert cost == case["cost"]
        assert [[list(b), l] for b, l in trace] == case["trace"]


@pytest.mark.parametrize("name,n", [("cfg1", 1 << 20), ("cfg2", 1 << 20), ("cfg3", 1 << 20), ("cfg4", 1 << 20),
                                    ("cfg5", 1 << 20)])
@pytest.mark.parametrize("k", [4, 2])
def test_recipes_vs_oracle(name, n, k, dev):
    keys = workloads.generate(name, n=n, seed=11)
    variant = "4way" if k == 4 else "2way"
    ref = oracle.sort(keys, k=k, variant=variant)
    out, perm, stats = gpu_sort(keys, dev, k=k, variant=variant)
    assert np.array_equal(perm, ref.values)
    assert np.array_equal(out.view(np.uint8), ref.keys.view(np.uint8))
    for f in POLICY_FIELDS + COUNTER_FIELDS:
        assert getattr(stats, f) == ref.stats[f], f
    assert stats.run_lengths == ref.run_lengths
    assert stats.natural_run_lengths == ref.natural_run_lengths
    assert read_trace(device=dev) == ref.trace
    assert scanned_elements_estimate(stats, n) == 4 * ref.stats["merge_cost"] + 2 * n


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("name,mrl", [("cfg1", 24), ("cfg2", 24), ("cfg3", 7), ("cfg4", 200), ("cfg5", 24)])
def test_counters_vs_oracle(name, mrl, variant, dev):
    # CountingOrder comparisons / moves and copy-smaller's buffer / scan counters
    # through the pipe kernel's stage sizes (statskit.py:49-98)
    n = 1 << 19
    keys = workloads.generate(name, n=n, seed=23)
    k = VARIANTS[variant]
    ref = oracle.sort(keys, k=k, variant=variant, min_run_len=mrl)
    out, perm, stats = gpu_sort(keys, dev, k=k, variant=variant, min_run_len=mrl, count_comparisons=True)
    assert np.array_equal(perm, ref.values)
    for f in POLICY_FIELDS + COUNTER_FIELDS + ("moves", "comparisons"):
        assert getattr(stats, f) == ref.stats[f], f
    _, _, plain = gpu_sort(keys, dev, k=k, variant=variant, min_run_len=mrl)
    for f in COUNTER_FIELDS:  # copy-smaller's counters without count_comparisons
        assert getattr(plain, f) == ref.stats[f], f


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_counters_adversarial_runs(variant, dev):
    # run ends far from the merged order of the other runs (long safe == 0
    # stretches of the stages kernels), heavy ties, single-record runs
    rng = np.random.default_rng(77)
    k = VARIANTS[variant]
    for trial in range(60):
        parts = []
        for _ in range(int(rng.integers(2, 40))):
            ln = int(rng.integers(1, 3000))
            kind = trial % 4
            if kind == 0:
                run = np.sort(rng.integers(0, 1 << 20, size=ln))
                run[-1] = (1 << 30) + int(rng.integers(0, 4))  # huge last record
            elif kind == 1:
                run = np.sort(rng.integers(0, 6, size=ln))  # ties
            elif kind == 2:
                run = np.sort(rng.integers(-(1 << 20), 1 << 20, size=ln))[::-1].copy()
                run[0] = -(1 << 30)  # breaks the descent: a short run then an ascent
            else:
                run = np.arange(ln) * 3 + int(rng.integers(0, 3))
            parts.append(run)
        keys = np.concatenate(parts).astype(np.int32)
        mrl = int(rng.choice([1, 2, 24, 100]))
        ref = oracle.sort(keys, k=k, variant=variant, min_run_len=mrl)
        _, perm, stats = gpu_sort(keys, dev, k=k, variant=variant, min_run_len=mrl, count_comparisons=True)
        assert np.array_equal(perm, ref.values), trial
        for f in POLICY_FIELDS + COUNTER_FIELDS + ("moves", "comparisons"):
            assert getattr(stats, f) == ref.stats[f], (f, trial)


def test_cfg1_full_matches_reference_golden(golden_cfg_full, dev):
    import hashlib

    g = golden_cfg_full["cfg1"]
    keys = workloads.generate("cfg1", n=g["n"], seed=g["seed"])
    out, perm, stats = gpu_sort(keys, dev)
    assert hashlib.sha256(perm.astype(np.int64).tobytes()).hexdigest() == g["perm_sha256"]
    for f in POLICY_FIELDS + COUNTER_FIELDS:
        assert getattr(stats, f) == g["stats"][f], f
    trace = read_trace(device=dev)
    flat = [x for b, l in trace for x in (len(b) - 1, *b, *([-1] * (5 - len(b))), l)]
    assert hashlib.sha256(np.asarray(flat, dtype=np.int64).tobytes()).hexdigest() == g["trace_sha256"]


@pytest.mark.parametrize("mrl", [1, 2, 7, 24, 64, 255, 256, 257, 600])
def test_min_run_len_sweep(mrl, dev):
    rng = np.random.default_rng(mrl)
    for kind in range(3):
        n = int(rng.integers(1, 40000))
        if kind == 0:
            keys = rng.integers(0, 50, size=n).astype(np.int32)
        elif kind == 1:
            keys = workloads.cfg2(n=n, seed=mrl)
        else:
            keys = np.sort(rng.integers(-100, 100, size=n)).astype(np.int64)
            keys[n // 3 : n // 2] = keys[n // 3 : n // 2][::-1]
        ref = oracle.sort(keys, min_run_len=mrl)
        out, perm, stats = gpu_sort(keys, dev, min_run_len=mrl)
        assert np.array_equal(perm, ref.values), (mrl, kind, n)
        assert stats.run_lengths == ref.run_lengths
        assert stats.merge_cost == ref.stats["merge_cost"]
        assert read_trace(device=dev) == ref.trace


@pytest.mark.parametrize("mrl", [5, 24, 200, 256])
def test_min_run_len_multilevel_chain_scan(mrl, dev):
    # > TSCAN_FAN groups of 16384 keys: the run-boundary chain scan goes
    # through compose/top/down levels (64 KB of staged tables at m = 256)
    n = 1_300_000 + 4 * mrl  # cfg4 needs n % 4 == 0
    keys = workloads.cfg4(n=n, seed=mrl)
    ref = oracle.sort(keys, min_run_len=mrl)
    out, perm, stats = gpu_sort(keys, dev, min_run_len=mrl)
    assert np.array_equal(perm, ref.values), mrl
    assert stats.run_lengths == ref.run_lengths
    assert stats.merge_cost == ref.stats["merge_cost"]


@pytest.mark.parametrize("mrl", [1025, 3000, 5000])
def test_min_run_len_beyond_tile_windows(mrl, dev):
    # windows longer than the formation tile's staging (1024): one CTA sorts each
    rng = np.random.default_rng(mrl)
    for kind in range(3):
        n = int(rng.integers(mrl, 60000))
        if kind == 0:
            keys = rng.integers(0, 50, size=n).astype(np.int32)
        elif kind == 1:
            keys = workloads.cfg2(n=n, seed=mrl)
        else:
            keys = rng.normal(size=n).astype(np.float64)
            keys[n // 4 : n // 2] = np.sort(keys[n // 4 : n // 2])[::-1]
        ref = oracle.sort(keys, min_run_len=mrl)
        out, perm, stats = gpu_sort(keys, dev, min_run_len=mrl)
        assert np.array_equal(perm, ref.values), (mrl, kind, n)
        assert np.array_equal(out.view(np.uint8), ref.keys.view(np.uint8))
        assert stats.run_lengths == ref.run_lengths
        assert stats.merge_cost == ref.stats["merge_cost"]
        assert read_trace(device=dev) == ref.trace


def test_values_payload_permuted(dev):
    keys_np = workloads.cfg3(n=1 << 16, seed=5)
    vals_np = np.random.default_rng(1).integers(-1000, 1000, size=keys_np.size).astype(np.int32)
    keys = torch.from_numpy(keys_np).to(dev)
    vals = torch.from_numpy(vals_np).to(dev)
    stable_sort_with(keys, SortConfig(), values=vals)
    perm = np.argsort(keys_np, kind="stable")
    assert np.array_equal(vals.cpu().numpy(), vals_np[perm])
    assert np.array_equal(keys.cpu().numpy(), keys_np[perm])


def test_unaligned_tensor_views(dev):
    # views at 4-byte offsets: the C ABI rejects them (TMA needs 16-byte
    # alignment), the Python entry point sorts aligned copies
    from paper_2209_06909_b200 import _lib

    base_np = workloads.cfg2(n=100_003, seed=2)
    full = torch.from_numpy(base_np).to(dev)
    view = full[1:]
    assert view.data_ptr() % 16 != 0
    out, perm, stats = stable_argsort(view, SortConfig())
    ref = oracle.sort(base_np[1:])
    assert np.array_equal(perm.cpu().numpy(), ref.values)
    vals = torch.zeros(view.numel(), dtype=torch.int32, device=dev)
    lib = _lib.load()
    cfg = _lib.PsConfig(4, 3, 24, 0, _lib.VALUES_ARGSORT)
    st = _lib.PsStats()
    ws = torch.empty(lib.ps_workspace_size(view.numel(), 0, cfg), dtype=torch.uint8, device=dev)
    rc = lib.ps_sort(0, view.data_ptr(), vals.data_ptr(), view.numel(), cfg, ws.data_ptr(), ws.numel(), st,
                     torch.cuda.current_stream(dev).cuda_stream)
    assert rc == 1  # PS_EINVAL


def test_list_api_records(dev):
    from operator import itemgetter

    rng = np.random.default_rng(3)
    keys = rng.integers(0, 7, size=300).tolist()
    records = [(k, i) for i, k in enumerate(keys)]
    lst = list(records)
    stats = stable_sort_with(lst, SortConfig(key=itemgetter(0)))
    assert lst == sorted(records, key=itemgetter(0))
    assert stats.runs_detected >= 1


def test_edge_sizes(dev):
    for n in (1, 2, 3, 23, 24, 25, 47, 48, 49, 2047, 2048, 2049, 16383, 16384, 16385, 16384 * 33 + 5):
        for gen in ("perm", "const", "desc", "asc"):
            if gen == "perm":
                keys = np.random.default_rng(n).permutation(n).astype(np.int32)
            elif gen == "const":
                keys = np.zeros(n, dtype=np.int32)
            elif gen == "desc":
                keys = np.arange(n, 0, -1).astype(np.int32)
            else:
                keys = np.arange(n).astype(np.int32)
            ref = oracle.sort(keys)
            out, perm, stats = gpu_sort(keys, dev)
            assert np.array_equal(perm, ref.values), (n, gen)
            assert stats.run_lengths == ref.run_lengths, (n, gen)
            assert stats.merge_cost == ref.stats["merge_cost"]


def test_unit_capacity_edges(dev):
    # nodes whose size or run lengths sit at the pipe kernel's unit capacities
    # (4-byte keys: 288 x 15 = 4320 records per unit, cuts every (4320 - 15) / arity;
    # 8-byte keys: 352 x 13 = 4576) and their multiples: one chunk exactly full,
    # one record more, runs one record around the cut spacing, and nodes that
    # fill a whole grid of units
    rng = np.random.default_rng(4320)

    def runs_of(lengths, dtype):
        parts = []
        for ln in lengths:
            v = np.sort(rng.integers(-(1 << 30), 1 << 30, ln)).astype(dtype)
            if ln:  # a descent between runs: every run ends high and starts low
                v[-1] = (1 << 30) + 7
                v[0] = -(1 << 30) - 7
            parts.append(v)
        return np.concatenate(parts)

    cases = []
    for cap, vt in ((4320, 15), (4576, 13)):
        cc = cap - vt
        for w in (2, 3, 4):
            s = cc // w
            for total in (cc - 1, cc, cc + 1, cap, cap + 1, 2 * cc, 2 * cc + 1):
                base = total // w
                cases.append([base] * (w - 1) + [total - base * (w - 1)])
            cases.append([s - 1, s, s + 1, 2 * s][:w])
            cases.append([2 * s, 2 * s + 1, 25, 4 * s][:w])
    cases.append([4320 * 74] * 4)      # 296 full units of one 4-way node
    cases.append([4305 * 74 + 1] * 4)
    for dtype in (np.int32, np.int64):
        for lengths in cases:
            keys = runs_of(lengths, dtype)
            ref = oracle.sort(keys)
            out, perm, stats = gpu_sort(keys, dev)
            assert np.array_equal(perm, ref.values), (dtype, lengths)
            assert stats.run_lengths == ref.run_lengths, (dtype, lengths)
            assert stats.merge_cost == ref.stats["merge_cost"], (dtype, lengths)


def test_float_signed_zero_and_ties(dev):
    rng = np.random.default_rng(9)
    keys = rng.choice(np.array([-0.0, 0.0, 1.0, -1.0, 2.5], dtype=np.float32), size=50000)
    ref = oracle.sort(keys)
    out, perm, stats = gpu_sort(keys, dev)
    assert np.array_equal(perm, ref.values)
    assert np.array_equal(out.view(np.uint32), ref.keys.view(np.uint32))


@pytest.mark.parametrize("name,n,mrl", [
    ("cfg1", 1 << 14, 24),    # r ~ 680: one-CTA tree, arrays in global memory
    ("cfg1", 1 << 17, 24),    # r ~ 5.5K: one-CTA tree, arrays in shared memory
    ("cfg4", 1 << 18, 24),    # r ~ 5.5K with the long ascending half
    ("cfg1", 1 << 18, 24),    # r ~ 11K: multi-kernel tree
    ("cfg1", 1 << 16, 8),     # network windows of 8
    ("cfg1", 1 << 16, 13),    # network windows of 16 (padded)
    ("cfg1", 1 << 16, 30),    # network windows of 32 (padded)
    ("cfg4", 1 << 16, 3),     # shortest fast-step windows
])
@pytest.mark.parametrize("dtype", ["int32", "float64"])
def test_tree_paths_and_windows(name, n, mrl, dtype, dev):
    keys = workloads.generate(name, n=n, seed=5)
    if dtype == "float64":
        keys = (keys.astype(np.float64) / 7.0).astype(np.float64)
    ref = oracle.sort(keys, k=4, variant="4way", min_run_len=mrl)
    out, perm, stats = gpu_sort(keys, dev, k=4, variant="4way", min_run_len=mrl)
    assert np.array_equal(perm, ref.values)
    assert np.array_equal(out.view(np.uint8), ref.keys.view(np.uint8))
    for f in POLICY_FIELDS + COUNTER_FIELDS:
        assert getattr(stats, f) == ref.stats[f], f
    assert stats.run_lengths == ref.run_lengths
    assert read_trace(device=dev) == ref.trace
    # a values payload through the network windows and the in-place leaves
    vals = torch.arange(n, dtype=torch.int32, device=dev) * 3 + 1
    kt = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    stable_sort_with(kt, SortConfig(min_run_len=mrl), values=vals)
    torch.cuda.synchronize()
    assert np.array_equal(vals.cpu().numpy(), ref.values * 3 + 1)


_TINY_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import oracle
from paper_2209_06909_b200 import SortConfig, stable_argsort, workloads
from paper_2209_06909_b200.policy import check
dev = torch.device('cuda', 0)
for name, n, dt, mrl in (('cfg4', 1 << 18, 'int32', 24), ('cfg1', 1 << 17, 'int32', 24), ('cfg1', 1 << 17, 'int64', 8),
                         ('cfg4', 1 << 16, 'float32', 3), ('cfg1', 1 << 16, 'int32', 2), ('cfg2', 1 << 20, 'int32', 24),
                         ('cfg3', 1 << 19, 'int64', 24), ('cfg5', 1 << 19, 'float32', 24)):
    keys = workloads.generate(name, n=n, seed=9).astype(dt)
    ref = oracle.sort(keys, min_run_len=mrl)
    out, perm, stats = stable_argsort(torch.from_numpy(keys).to(dev), SortConfig(min_run_len=mrl))
    check(dev)
    assert np.array_equal(perm.cpu().numpy(), ref.values), (name, dt, mrl)
    assert np.array_equal(out.cpu().numpy().view(np.uint8), ref.keys.view(np.uint8)), (name, dt, mrl)
    assert stats.merge_cost == ref.stats['merge_cost']
print('TINY OK')
"""


def test_tiny_node_kernel_and_thin_partition_forced(dev):
    # the thread-per-node merge runs only on stages with >= 32K small nodes and
    # the thin partition only on stages with >= 12K cuts; PS_TINY_MIN=1 and
    # PS_THIN_CUTS=1 (read once per process) force them onto every stage
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # the knobs are read only by the measurement build (-DPS_DEBUG_KNOBS)
    sys.path.insert(0, repo)
    import __graft_entry__

    debug_lib = __graft_entry__.build_lib(debug=True)
    env = dict(os.environ, PS_TINY_MIN="1", PS_THIN_CUTS="1", PS_LIB=debug_lib)
    r = subprocess.run([sys.executable, "-c", _TINY_SCRIPT, repo], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "TINY OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("shape,dtype", [((), torch.int64), ((3,), torch.float64), ((5,), torch.uint8),
                                         ((2, 3), torch.float32), ((), torch.int16)])
def test_payload_rows_any_width(shape, dtype, dev):
    # payloads wider or narrower than int32 follow the stable permutation (ps_gather_rows)
    n = 40001
    keys_np = workloads.generate("cfg3", n=n, seed=4)
    order = np.argsort(keys_np, kind="stable")
    vals = torch.arange(n * int(np.prod(shape, dtype=np.int64)), device=dev).reshape((n,) + shape).to(dtype)
    want = vals.cpu().numpy()[order]
    keys = torch.from_numpy(keys_np).to(dev)
    stats = stable_sort_with(keys, SortConfig(), values=vals)
    torch.cuda.synchronize()
    assert np.array_equal(keys.cpu().numpy(), keys_np[order])
    assert np.array_equal(vals.cpu().numpy(), want)
    assert stats.merge_cost > 0


def test_concurrent_sorts_on_two_streams(dev):
    # the reference allows concurrent sorts: two host threads,
    # each with its own stream (and so its own workspace), sorting at once;
    # the fused-partition pipe launches are cooperative, so neither starves
    # the other's grid barrier
    import threading

    inputs = [workloads.generate("cfg2", n=1 << 22, seed=41), workloads.generate("cfg3", n=1 << 21, seed=42),
              workloads.generate("cfg5", n=1 << 22, seed=43), workloads.generate("cfg1", n=1 << 20, seed=44)]
    refs = [oracle.sort(x, want_trace=False) for x in inputs]
    errors = []

    def worker(idx):
        try:
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                for rep in range(6):
                    x = inputs[(idx + 2 * rep) % len(inputs)]
                    ref = refs[(idx + 2 * rep) % len(inputs)]
                    keys = torch.from_numpy(x).to(dev)
                    out, perm, _ = stable_argsort(keys, SortConfig())
                    s.synchronize()
                    if not np.array_equal(perm.cpu().numpy(), ref.values):
                        errors.append((idx, rep))
        except Exception as e:  # noqa: BLE001
            errors.append((idx, repr(e)))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_asynchronous_sorts_then_check(dev):
    # PS_FLAG_ASYNC: ps_sort returns with the merges queued; check() reports
    # their device invariants afterwards
    from paper_2209_06909_b200 import _lib
    from paper_2209_06909_b200.policy import _sort_tensor, check

    streams = [torch.cuda.Stream(dev) for _ in range(2)]
    work = []
    for i, s in enumerate(streams):
        x = workloads.generate("cfg2", n=1 << 21, seed=60 + i)
        with torch.cuda.stream(s):
            keys = torch.from_numpy(x).to(dev)
            perm = torch.empty(x.shape[0], dtype=torch.int32, device=dev)
            _sort_tensor(keys, perm, SortConfig(count_comparisons=False), _lib.VALUES_ARGSORT, collect_runs=False,
                         asynchronous=True)
        work.append((x, s, keys, perm))
    for x, s, keys, perm in work:
        with torch.cuda.stream(s):
            check(dev)
        assert np.array_equal(perm.cpu().numpy(), oracle.sort(x, want_trace=False).values)


@pytest.mark.parametrize("name,k", [("cfg2", 4), ("cfg4", 4), ("cfg1", 2)])
def test_asynchronous_counting_sort_then_finish_counters(name, k, dev):
    # PS_FLAG_ASYNC with the counters on: comparisons / moves stay on the device
    # (ps_stats.*_valid == 2) until finish_counters() reads them after the stream
    from paper_2209_06909_b200 import _lib
    from paper_2209_06909_b200.policy import _sort_tensor, finish_counters

    x = workloads.generate(name, n=1 << 20, seed=71)
    variant = "4way" if k == 4 else "2way"
    keys = torch.from_numpy(x).to(dev)
    perm = torch.empty(x.shape[0], dtype=torch.int32, device=dev)
    st = _sort_tensor(keys, perm, SortConfig(k=k, variant=variant), _lib.VALUES_ARGSORT, collect_runs=False,
                      asynchronous=True)
    assert st.comparisons is None and st.moves is None
    finish_counters(st)
    ref = oracle.sort(x, k=k, variant=variant, want_trace=False)
    assert st.comparisons == ref.stats["comparisons"] and st.moves == ref.stats["moves"]
    assert np.array_equal(perm.cpu().numpy(), ref.values)
