"""The reference's own test suite, unmodified, against the B200 package.

``compat/powersort`` is a ``powersort`` package whose sort entry points are
``paper_2209_06909_b200``'s.  These tests run the
reference's test modules for the public surface -- test_policy.py (the sort:
anchors, hand-traced schedules, merge_down arities, stability on records,
SENTINEL fallback, simulator == real trace, k=2 strict tree), test_statskit.py,
test_power.py and test_acceptance.py (the 10,000-trial correctness and
stability matrix over every variant, generator and min_run_len, the
merge-cost, comparison and stack-height theorems, oracle dominance,
near-optimality, merge-cost halving, scanned-element consistency, trivial
anchors) -- in a subprocess with ``compat/`` first on sys.path, so every
``stable_sort_with`` they call sorts on the GPU.

The reference sources are staged by tools/stage_reference.sh into the
git-ignored ``baseline/_ref`` (installed package + a copy of its tests); the
tests skip when that staging is absent.  Nothing here reads /root/reference.
"""

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")


def _run_suite(files, extra=()):
    if not (os.path.isdir(os.path.join(REF, "powersort")) and os.path.isdir(REF_TESTS)):
        pytest.skip("reference suite not staged (run tools/stage_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REPO, "compat"), REPO, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", REF_TESTS, "-c",
           os.devnull] + [os.path.join(REF_TESTS, f) for f in files] + list(extra)
    res = subprocess.run(cmd, env=env, cwd=REF_TESTS, capture_output=True, text=True, timeout=1800)
    tail = (res.stdout + res.stderr)[-4000:]
    assert res.returncode == 0, tail
    # the shim really served the sort from the B200 package
    assert " passed" in res.stdout, tail
    return res.stdout


def test_shim_serves_the_b200_package():
    if not os.path.isdir(os.path.join(REF, "powersort")):
        pytest.skip("reference package not staged (run tools/stage_reference.sh)")
    code = ("import powersort, paper_2209_06909_b200 as p;"
            "assert powersort.stable_sort_with is p.stable_sort_with;"
            "assert powersort.policy.merge_cost_for_profile is p.merge_cost_for_profile;"
            "assert powersort.SortConfig is p.SortConfig;"
            "assert powersort.node_power is p.node_power;"
            "assert powersort.oracle.__name__.startswith('_powersort_ref');"
            "print('ok')")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REPO, "compat"), REPO, env.get("PYTHONPATH", "")])
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_reference_power_suite():
    # node_power / run_stack_capacity / boundary_powers through the C ABI (host code)
    _run_suite(["test_power.py"])


@pytest.mark.gpu
def test_reference_policy_suite():
    _run_suite(["test_policy.py"])


@pytest.mark.gpu
def test_reference_statskit_suite():
    _run_suite(["test_statskit.py"])


@pytest.mark.gpu
def test_reference_acceptance_suite():
    # the reference's acceptance criteria, every stable_sort_with on the GPU
    out = _run_suite(["test_acceptance.py"])
    assert " failed" not in out
