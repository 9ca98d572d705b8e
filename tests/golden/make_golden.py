"""Generate the golden parity fixtures by running the REFERENCE itself.

Imports the read-only Python reference from /root/reference/pkg/src (only
available in the build container, never on the GPU box) and records, for
seeded inputs, exactly what ``stable_sort_with`` / ``merge_cost_for_profile``
/ ``node_power`` return: the stable permutation, every SortStats counter,
run_lengths, natural_run_lengths and the on_merge trace.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed): tests/golden/sorts.json.gz, profiles.json.gz,
powers.json.gz, cfg_full.json (its "seconds" field is the reference's run
time).  Regenerating must reproduce the rest bit for bit.  ``make_golden.py
harness`` writes only tests/golden/harness.json: the reference harness's
generator outputs and per-trial seeds.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys
import time
from operator import itemgetter

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, REPO)

import powersort  # noqa: E402  (the reference)
from powersort.policy import SortConfig, merge_cost_for_profile, stable_sort_with  # noqa: E402
from powersort.power import _node_power_any, node_power, run_stack_capacity  # noqa: E402

from paper_2209_06909_b200 import workloads  # noqa: E402

VARIANTS = ["2way", "2way-copy-smaller", "2way-nosentinel", "4way", "4way-nosentinel"]
K_OF = {"2way": 2, "2way-copy-smaller": 2, "2way-nosentinel": 2, "4way": 4, "4way-nosentinel": 4}
STAT_FIELDS = ["comparisons", "merge_cost", "buffer_cost", "moves", "max_stack_height", "runs_detected",
               "merges2", "merges3", "merges4", "scan_reads", "scan_writes"]


def ref_sort(keys, variant, min_run_len, strict):
    """Reference stable_sort_with on (key, index) records."""
    records = [(k, i) for i, k in enumerate(keys)]
    trace = []
    cfg = SortConfig(k=K_OF[variant], variant=variant, min_run_len=min_run_len, key=itemgetter(0),
                     strict_merge_down=strict, on_merge=trace.append)
    stats = stable_sort_with(records, cfg)
    perm = [i for _, i in records]
    return perm, stats, trace


def stats_dict(stats):
    d = {f: int(getattr(stats, f)) for f in STAT_FIELDS}
    d["run_lengths"] = list(stats.run_lengths)
    d["natural_run_lengths"] = list(stats.natural_run_lengths)
    return d


def trace_list(trace):
    return [[list(b), int(length)] for b, length in trace]


def gen_keys(rng, kind, n):
    """Small inputs covering the semantic edge cases."""
    if kind == "dup":
        return [rng.randint(0, rng.choice([1, 2, 7, 127])) for _ in range(n)]
    if kind == "perm":
        xs = list(range(n))
        rng.shuffle(xs)
        return xs
    if kind == "runs":
        out = []
        while len(out) < n:
            length = rng.randint(1, 60)
            seg = sorted(rng.randint(-50, 50) for _ in range(length))
            if rng.random() < 0.5:
                seg = seg[::-1]
            out.extend(seg)
        return out[:n]
    if kind == "sorted":
        return list(range(n))
    if kind == "reverse":
        return list(range(n, 0, -1))
    if kind == "plateaus":
        out = []
        while len(out) < n:
            v = rng.randint(0, 5)
            out.extend([v] * rng.randint(1, 30))
        return out[:n]
    if kind == "float":
        vals = [rng.choice([-0.0, 0.0, 1.5, -2.25, 3.0, float(rng.randint(-9, 9)) / 4]) for _ in range(n)]
        return [float(np.float32(v)) for v in vals]
    if kind == "int64":
        pal = [rng.randint(-(2**62), 2**62) for _ in range(rng.randint(1, 12))]
        return [rng.choice(pal) for _ in range(n)]
    raise ValueError(kind)


def make_sorts():
    rng = random.Random(20240917)
    cases = []
    kinds = ["dup", "perm", "runs", "sorted", "reverse", "plateaus", "float", "int64"]
    for variant in VARIANTS:
        for mrl in (1, 2, 3, 5, 24, 40):
            for strict in (False, True):
                for kind in kinds:
                    n = rng.choice([0, 1, 2, 3, 5, 17, 24, 25, 48, 97, 200, 511, 1200])
                    keys = gen_keys(rng, kind, n)
                    dtype = "float32" if kind == "float" else ("int64" if kind == "int64" else "int32")
                    perm, stats, trace = ref_sort(keys, variant, mrl, strict)
                    cases.append({
                        "keys": keys, "dtype": dtype, "variant": variant, "k": K_OF[variant],
                        "min_run_len": mrl, "strict": strict, "perm": perm,
                        "stats": stats_dict(stats), "trace": trace_list(trace),
                    })
    # bigger ones, default config (k=4, "4way", mrl 24) on the cfg recipes at small n
    for name, n in (("cfg1", 4096), ("cfg2", 16384), ("cfg3", 16384), ("cfg4", 16384), ("cfg5", 8192)):
        keys = workloads.generate(name, n=n, seed=1).tolist()
        for variant, strict in (("4way", False), ("2way", False), ("4way", True)):
            perm, stats, trace = ref_sort(keys, variant, 24, strict)
            cases.append({
                "keys": keys, "dtype": {"cfg3": "int64", "cfg5": "float32"}.get(name, "int32"),
                "variant": variant, "k": K_OF[variant], "min_run_len": 24, "strict": strict, "perm": perm,
                "stats": stats_dict(stats), "trace": trace_list(trace), "recipe": name,
            })
    return cases


def make_profiles():
    rng = random.Random(99)
    out = []
    for _ in range(400):
        r = rng.randint(1, 40)
        prof = [rng.randint(2, 200) for _ in range(r - 1)] + [rng.randint(1, 200)]
        for k in (2, 4):
            for strict in (False, True):
                tr = []
                cost = merge_cost_for_profile(prof, k, strict_merge_down=strict, on_merge=tr.append)
                out.append({"lengths": prof, "k": k, "strict": strict, "cost": cost, "trace": trace_list(tr)})
    # the reference tests' hand-traced profiles
    for prof in ([2, 2, 4, 8], [4, 4, 4, 4, 48], [4, 2, 2, 8], [16, 8, 4, 2, 1], [32, 16, 8, 4, 2, 1],
                 [2 ** (8 - i) for i in range(9)], [24] * 1000):
        for k in (2, 4):
            for strict in (False, True):
                tr = []
                cost = merge_cost_for_profile(prof, k, strict_merge_down=strict, on_merge=tr.append)
                out.append({"lengths": prof, "k": k, "strict": strict, "cost": cost, "trace": trace_list(tr)})
    return out


def make_powers():
    rng = random.Random(7)
    out = []
    for _ in range(3000):
        n = rng.choice([2, 3, 10, 1000, 10**6, 2**24, 2**31, 2**31 - 1, 10**8, 2**40])
        e2 = rng.randint(3, n) if n >= 3 else n
        b1 = rng.randint(0, e2 - 2)
        e1 = rng.randint(b1 + 1, e2 - 1)
        k = rng.choice([2, 3, 4])
        out.append([k, n, b1, e1, e1, e2, _node_power_any(k, n, b1, e1, e1, e2)])
    caps = [[k, n, run_stack_capacity(k, n)] for k in (2, 3, 4) for n in (1, 2, 16, 10**6, 2**24, 2**31)]
    return {"powers": out, "caps": caps, "node_power_2_4": node_power(2, 4, 0, 2, 2, 4)}


def sha(arr):
    return hashlib.sha256(np.asarray(arr, dtype=np.int64).tobytes()).hexdigest()


def make_cfg_full():
    """Full-size cfg1 through the reference (about 10 s), recorded as hashes."""
    out = {}
    for name, n in (("cfg1", 2**20),):
        keys = workloads.generate(name, n=n, seed=0)
        t = time.time()
        perm, stats, trace = ref_sort(keys.tolist(), "4way", 24, False)
        dt = time.time() - t
        flat = [x for b, length in trace for x in (len(b) - 1, *b, *([-1] * (5 - len(b))), length)]
        out[name] = {
            "n": n, "seed": 0, "seconds": dt, "perm_sha256": sha(perm),
            "stats": {f: int(getattr(stats, f)) for f in STAT_FIELDS},
            "run_lengths_sha256": sha(stats.run_lengths),
            "natural_run_lengths_sha256": sha(stats.natural_run_lengths),
            "trace_sha256": sha(flat), "trace_len": len(trace),
            "keys_sha256": hashlib.sha256(keys.tobytes()).hexdigest(),
        }
    return out


def dump(name, obj):
    path = os.path.join(HERE, name)
    data = json.dumps(obj, separators=(",", ":")).encode()
    if name.endswith(".gz"):
        with gzip.GzipFile(path, "wb", mtime=0) as f:
            f.write(data)
    else:
        with open(path, "wb") as f:
            f.write(json.dumps(obj, indent=1).encode())
    print(name, len(data), "bytes")


def make_harness():
    # the reference harness's generators and per-trial seeds (harness.py:74-134),
    # for the GPU harness's restatement (paper_2209_06909_b200/harness.py)
    from powersort import harness as rh

    cases = []
    for kind, n, exp in (("random-runs", 1000, None), ("random-runs", 4099, 7), ("random-runs", 20000, 1),
                         ("random-runs", 50000, 300), ("random-permutation", 3000, None), ("sorted", 77, None),
                         ("reverse", 77, None)):
        for base, trial in ((0, 0), (3, 1), (12345, 2)):
            seed = rh.derive_seed(base, trial)
            arr = np.asarray(rh.generate(rh.GeneratorSpec(kind, n, expected_run_len=exp, seed=seed)),
                             dtype=np.int64)
            cases.append({"kind": kind, "n": n, "expected_run_len": exp, "base": base, "trial": trial,
                          "seed": seed, "sha": sha(arr), "head": arr[:8].tolist()})
    return {"csv_header": rh.CSV_HEADER, "cases": cases}


if __name__ == "__main__":
    assert os.path.isdir(REF), "the reference is only present in the build container"
    if sys.argv[1:] == ["harness"]:
        dump("harness.json", make_harness())
        sys.exit(0)
    print("reference powersort", powersort.__version__)
    dump("sorts.json.gz", make_sorts())
    dump("profiles.json.gz", make_profiles())
    dump("powers.json.gz", make_powers())
    dump("cfg_full.json", make_cfg_full())
