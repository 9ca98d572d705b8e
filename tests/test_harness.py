"""The GPU benchmark CLI (paper_2209_06909_b200.harness): its generators and
seeds against the reference harness's own output (tests/golden/harness.json),
and its CSV rows against the oracle on the GPU."""

import csv
import hashlib
import io
import json
import os

import numpy as np
import pytest

from paper_2209_06909_b200 import harness

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "harness.json")


def _sha(arr):
    return hashlib.sha256(np.asarray(arr, dtype=np.int64).tobytes()).hexdigest()


def test_generators_and_seeds_match_reference():
    g = json.load(open(GOLDEN))
    assert harness.CSV_HEADER == g["csv_header"]
    for c in g["cases"]:
        seed = harness.derive_seed(c["base"], c["trial"])
        assert seed == c["seed"], c
        arr = harness.generate(c["kind"], c["n"], seed, c["expected_run_len"])
        assert arr[:8].tolist() == c["head"], c
        assert _sha(arr) == c["sha"], c


def test_run_entropy():
    assert harness.run_entropy([5]) == 0.0
    assert harness.run_entropy([1, 1, 1, 1]) == pytest.approx(2.0, abs=1e-12)
    assert harness.run_entropy([2, 6]) == pytest.approx(0.8112781244591328, abs=1e-12)


def test_cli_rejects_unknown_ids():
    with pytest.raises(SystemExit):
        harness.main(["--algo", "gpu-9way", "--input", "sorted", "--n", "10", "--trials", "1", "--seed", "0"])


@pytest.mark.gpu
def test_cli_rows_match_oracle(tmp_path):
    from oracle import oracle

    out = tmp_path / "rows.csv"
    rc = harness.main(["--algo", "gpu-4way,gpu-2way,4way-nosentinel", "--input", "random-runs", "--n", "6000",
                       "--expected-run-len", "9", "--trials", "2", "--seed", "7", "--elem", "record",
                       "--csv", str(out)])
    assert rc == 0
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    assert len(rows) == 6 and ",".join(rows[0].keys()) == harness.CSV_HEADER
    for row in rows:
        variant = row["algo"][4:]
        k = 4 if variant.startswith("4way") else 2
        keys = harness.generate("random-runs", 6000, int(row["seed"]), 9)
        ref = oracle.sort(keys, k=k, variant=variant)
        for col, f in (("merge_cost", "merge_cost"), ("buffer_cost", "buffer_cost"), ("runs", "runs_detected"),
                       ("max_stack", "max_stack_height"), ("merges2", "merges2"), ("merges3", "merges3"),
                       ("merges4", "merges4"), ("comparisons", "comparisons"), ("moves", "moves")):
            assert int(row[col]) == ref.stats[f], (row["algo"], col)
        assert int(row["scanned_estimate"]) == 4 * ref.stats["merge_cost"] + 2 * 6000
        assert float(row["entropy_bits"]) == pytest.approx(harness.run_entropy(ref.run_lengths), abs=1e-9)
        assert int(row["time_ns"]) > 0
