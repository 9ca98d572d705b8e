"""GPU counterpart of the reference's ``powersort-bench`` CLI.

Same options, same input generators and per-trial seeds, and the same CSV
header as the reference harness (``harness.py:50-53``), so GPU rows sit next
to the reference's CPU rows and can be compared pairwise by existing tooling.
Algorithm ids are the reference's merge variants prefixed with ``gpu-``
(``gpu-4way`` ...); the plain ids are accepted too and mean the same GPU sort.

The generators restate the reference's published recipes (``harness.py:74-134``):
numpy PCG64 seeded with ``SeedSequence(seed)``; per-trial seed
``SeedSequence((base, trial)).generate_state(1, uint64)[0]``; random-runs =
geometric run lengths (p = 1 / expected length, default isqrt(n)) truncated to
n, keys uniform in [0, 2^31) sorted per run, each run shifted down to start
strictly below the previous run's last key.  tests/golden/harness.json pins
them to the reference's own output.

Columns:
* time_ns -- device time of one sort with the keys resident on the GPU (CUDA
  events around ``ps_sort`` and its merges), not Python-list time;
* comparisons / moves -- the reference's CountingOrder counts, from a second,
  counting sort of the same input (``SortConfig.count_comparisons``);
* every other counter and entropy_bits (of the run-length profile,
  ``oracle.py:111-122``) as the reference reports them.

usage: python -m paper_2209_06909_b200.harness --algo gpu-4way --input random-runs \\
           --n 1e6 --trials 3 --seed 1 [--elem record] [--csv out.csv]
"""

from __future__ import annotations

import argparse
import math
import sys

import numpy as np

GENERATOR_KINDS = ("random-runs", "random-permutation", "sorted", "reverse")
VARIANT_IDS = ("2way", "2way-copy-smaller", "2way-nosentinel", "4way", "4way-nosentinel")
ALGORITHMS = tuple("gpu-" + v for v in VARIANT_IDS) + VARIANT_IDS
MEASURES = ("time", "mergecost", "comparisons", "scanned")
CSV_HEADER = (
    "algo,n,seed,trial,time_ns,comparisons,merge_cost,buffer_cost,moves,"
    "max_stack,runs,merges2,merges3,merges4,scanned_estimate,entropy_bits"
)
KEY_RANGE = 1 << 31


def derive_seed(base_seed: int, trial: int) -> int:
    """Per-trial 64-bit seed: the (base, trial) split of numpy's SeedSequence."""
    return int(np.random.SeedSequence((base_seed, trial)).generate_state(1, dtype=np.uint64)[0])


def _run_lengths(rng, n: int, expected: int):
    # geometric lengths >= 1, drawn in batches, the last one cut to reach n
    p = 1.0 / expected
    batch = max(16, int(n / expected * 1.2) + 1)
    out, total = [], 0
    while total < n:
        draw = rng.geometric(p, size=batch)
        csum = np.cumsum(draw)
        stop = int(np.searchsorted(csum, n - total))  # first index reaching n - total
        if stop < len(draw):
            out.extend(int(x) for x in draw[:stop])
            out.append(n - total - (int(csum[stop - 1]) if stop else 0))
            total = n
        else:
            out.extend(int(x) for x in draw)
            total += int(csum[-1])
    return out


def generate(kind: str, n: int, seed: int, expected_run_len: int | None = None) -> np.ndarray:
    """int64 keys of one input (the reference's generator recipes)."""
    if n < 1:
        raise ValueError("generator needs n >= 1")
    if kind == "sorted":
        return np.arange(n, dtype=np.int64)
    if kind == "reverse":
        return np.arange(n - 1, -1, -1, dtype=np.int64)
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    if kind == "random-permutation":
        return rng.permutation(n).astype(np.int64)
    if kind == "random-runs":
        expected = expected_run_len if expected_run_len is not None else max(1, math.isqrt(n))
        if expected < 1:
            raise ValueError("expected_run_len must be >= 1")
        lengths = _run_lengths(rng, n, expected)
        keys = rng.integers(0, KEY_RANGE, size=n, dtype=np.int64)
        out = np.empty(n, dtype=np.int64)
        pos, tail = 0, None
        for ln in lengths:
            seg = np.sort(keys[pos:pos + ln])
            if tail is not None and seg[0] >= tail:
                seg = seg - (int(seg[0]) - tail + 1)  # a strict descent at the boundary
            out[pos:pos + ln] = seg
            tail = int(seg[-1])
            pos += ln
        return out
    raise ValueError("unknown generator kind %r (choose from %s)" % (kind, ", ".join(GENERATOR_KINDS)))


def run_entropy(lengths) -> float:
    """Entropy (bits) of the run-length fractions: lg n - (1/n) sum L lg L."""
    if len(lengths) <= 1:
        return 0.0
    n = sum(lengths)
    return math.log2(n) - math.fsum(ln * math.log2(ln) for ln in lengths) / n


def run_trial(algo: str, kind: str, n: int, base_seed: int, trial: int, min_run_len: int = 24,
              elem: str = "int", expected_run_len: int | None = None, device=None):
    """Generate, sort on the GPU, time, verify; returns (csv row dict, error or None)."""
    import torch

    from . import SortConfig, scanned_elements_estimate, stable_argsort
    from .policy import check

    variant = algo[4:] if algo.startswith("gpu-") else algo
    if variant not in VARIANT_IDS:
        raise ValueError("unknown algorithm %r" % algo)
    k = 4 if variant.startswith("4way") else 2
    dev = device or torch.device("cuda", 0)
    seed = derive_seed(base_seed, trial)
    keys_np = generate(kind, n, seed, expected_run_len)
    src = torch.from_numpy(keys_np).to(dev)
    cfg = SortConfig(k=k, variant=variant, min_run_len=min_run_len)
    keys = src.clone()
    stable_argsort(keys, cfg)  # warm-up (workspace, first-launch costs)
    keys = src.clone()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out, perm, stats = stable_argsort(keys, cfg)
    b.record()
    check(dev)
    torch.cuda.synchronize()
    time_ns = int(round(a.elapsed_time(b) * 1e6))
    _, _, cst = stable_argsort(src.clone(), SortConfig(k=k, variant=variant, min_run_len=min_run_len,
                                                     count_comparisons=True))
    # verification: the output is a permutation of the input, sorted, and (records)
    # equal keys keep their input order
    o = out.cpu().numpy()
    p = perm.cpu().numpy().astype(np.int64)
    error = None
    if not np.array_equal(np.sort(p), np.arange(n)) or not np.array_equal(keys_np[p], o):
        error = "output is not a permutation of the input"
    elif n > 1 and (o[1:] < o[:-1]).any():
        error = "output is not sorted (position %d)" % int(np.argmax(o[1:] < o[:-1]))
    elif elem == "record" and n > 1:
        tie = (o[1:] == o[:-1]) & (p[1:] < p[:-1])
        if tie.any():
            error = "equal keys out of input order (position %d)" % int(np.argmax(tie))
    row = {
        "algo": "gpu-" + variant,
        "n": n,
        "seed": seed,
        "trial": trial,
        "time_ns": time_ns,
        "comparisons": cst.comparisons,
        "merge_cost": stats.merge_cost,
        "buffer_cost": stats.buffer_cost,
        "moves": cst.moves,
        "max_stack": stats.max_stack_height,
        "runs": stats.runs_detected,
        "merges2": stats.merges2,
        "merges3": stats.merges3,
        "merges4": stats.merges4,
        "scanned_estimate": scanned_elements_estimate(stats, n),
        "entropy_bits": run_entropy(stats.run_lengths) if stats.run_lengths else 0.0,
    }
    return row, error


def write_csv(rows, fh):
    fh.write(CSV_HEADER + "\n")
    cols = CSV_HEADER.split(",")
    for row in rows:
        fh.write(",".join(("%.12g" % row[c]) if c == "entropy_bits" else str(row[c]) for c in cols) + "\n")


def _count(text):
    value = int(float(text))
    if value < 1:
        raise argparse.ArgumentTypeError("expected a positive count")
    return value


def main(argv=None):
    ap = argparse.ArgumentParser(prog="powersort-bench-gpu", description="Benchmark the B200 stable sorts.")
    ap.add_argument("--algo", required=True, help="comma-separated ids: %s" % ", ".join(ALGORITHMS))
    ap.add_argument("--input", required=True, choices=GENERATOR_KINDS)
    ap.add_argument("--n", required=True, type=_count, help="input size (accepts 1e6 style)")
    ap.add_argument("--expected-run-len", type=_count, default=None)
    ap.add_argument("--trials", required=True, type=_count)
    ap.add_argument("--seed", required=True, type=int)
    ap.add_argument("--min-run-len", type=_count, default=24)
    ap.add_argument("--measure", default=",".join(MEASURES), help="accepted for compatibility; all are collected")
    ap.add_argument("--elem", choices=("int", "record"), default="int")
    ap.add_argument("--csv", default="-")
    args = ap.parse_args(argv)
    for m in args.measure.split(","):
        if m and m not in MEASURES:
            ap.error("unknown measure %r" % m)
    algos = [a for a in args.algo.split(",") if a]
    for a in algos:
        if a not in ALGORITHMS:
            ap.error("unknown algorithm %r" % a)
    rows, errors = [], []
    for a in algos:
        for t in range(args.trials):
            row, err = run_trial(a, args.input, args.n, args.seed, t, args.min_run_len, args.elem,
                                 args.expected_run_len)
            rows.append(row)
            if err:
                errors.append("%s trial %d: %s" % (row["algo"], t, err))
    if args.csv == "-":
        write_csv(rows, sys.stdout)
    else:
        with open(args.csv, "w") as fh:
            write_csv(rows, fh)
    for e in errors:
        print("verification failure: %s" % e, file=sys.stderr)
    return 1 if errors else 0


if __name__ == "__main__":
    sys.exit(main())
