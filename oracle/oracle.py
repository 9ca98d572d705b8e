"""CPU oracle for the Multiway Powersort hot path -- TEST INFRASTRUCTURE ONLY.

This module wraps ``oracle/_build/libpsoracle.so``, a single-threaded C++
restatement of the reference ``powersort`` package
(``/root/reference/pkg/src/powersort``; see ``powersort_oracle.cpp`` for the
per-function file:line citations).  It is the parity checker: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it.  The product package
``paper_2209_06909_b200`` never imports it and has no CPU fallback.

Parity pin: the restatement is checked against golden vectors produced by the
Python reference itself (``tests/golden/make_golden.py`` ->
``tests/golden/*.json``) in ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libpsoracle.so")

VARIANT_IDS = {
    "2way": 0,
    "2way-copy-smaller": 1,
    "2way-nosentinel": 2,
    "4way": 3,
    "4way-nosentinel": 4,
}
VARIANT_K = {"2way": 2, "2way-copy-smaller": 2, "2way-nosentinel": 2, "4way": 4, "4way-nosentinel": 4}
DTYPE_IDS = {np.dtype(np.int32): 0, np.dtype(np.int64): 1, np.dtype(np.float32): 2, np.dtype(np.float64): 3}
STAT_FIELDS = (
    "comparisons",
    "merge_cost",
    "buffer_cost",
    "moves",
    "max_stack_height",
    "runs_detected",
    "merges2",
    "merges3",
    "merges4",
    "scan_reads",
    "scan_writes",
)


class _Stats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in STAT_FIELDS]


_lib = None


def build():
    """Compile the oracle (g++, seconds).  Called by __graft_entry__.build()."""
    subprocess.check_call(["make", "-s", "-C", _HERE])


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        lib.pso_sort.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
            ctypes.c_int64, ctypes.c_int, ctypes.POINTER(_Stats), ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int64, i64p,
        ]
        lib.pso_sort.restype = ctypes.c_int
        lib.pso_merge_cost_for_profile.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, i64p, i64p, ctypes.c_void_p,
            ctypes.c_int64, i64p,
        ]
        lib.pso_merge_cost_for_profile.restype = ctypes.c_int
        lib.pso_node_power.argtypes = [ctypes.c_int] + [ctypes.c_int64] * 5 + [ctypes.c_int]
        lib.pso_node_power.restype = ctypes.c_int
        lib.pso_run_stack_capacity.argtypes = [ctypes.c_int64, ctypes.c_int64]
        lib.pso_run_stack_capacity.restype = ctypes.c_int64
        lib.pso_detect_runs.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        lib.pso_detect_runs.restype = ctypes.c_int64
        _lib = lib
    return _lib


def _raise(code):
    if code == 1:
        raise ValueError("oracle: invalid argument")
    if code == 5:
        raise OverflowError("oracle: run stack exceeded its height bound")
    if code == 4:
        raise AssertionError("oracle: invariant violated")
    if code != 0:
        raise RuntimeError("oracle: error %d" % code)


@dataclass
class OracleResult:
    keys: np.ndarray
    values: np.ndarray
    stats: dict
    run_lengths: list = field(default_factory=list)
    natural_run_lengths: list = field(default_factory=list)
    trace: list = field(default_factory=list)  # [((b0, .., end), length), ...] like on_merge


def trace_rows_to_list(rows):
    out = []
    for row in rows:
        w = int(row[0])
        bounds = tuple(int(x) for x in row[1 : 2 + w])
        out.append((bounds, int(row[6])))
    return out


def sort(keys, values=None, k=4, variant="4way", min_run_len=24, strict_merge_down=False, want_trace=True,
         want_runs=True):
    """Stable sort of ``keys`` (copy) carrying ``values`` (default: the
    original index), exactly as ``stable_sort_with`` on (key, value) records
    with ``key=itemgetter(0)``.  Returns an OracleResult."""
    lib = _load()
    keys = np.ascontiguousarray(np.array(keys, copy=True))
    if keys.dtype not in DTYPE_IDS:
        raise ValueError("unsupported dtype %s" % keys.dtype)
    n = keys.shape[0]
    if values is None:
        values = np.arange(n, dtype=np.int32)
    values = np.ascontiguousarray(np.array(values, dtype=np.int32, copy=True))
    st = _Stats()
    runs = np.zeros(max(n, 1), dtype=np.int64) if want_runs else None
    nat = np.zeros(max(n, 1), dtype=np.int64) if want_runs else None
    cap = max(n, 1) if want_trace else 0
    rows = np.zeros((cap, 7), dtype=np.int64) if want_trace else None
    count = ctypes.c_int64(0)
    code = lib.pso_sort(
        DTYPE_IDS[keys.dtype], keys.ctypes.data, values.ctypes.data, n, k, VARIANT_IDS.get(variant, 99),
        min_run_len, int(bool(strict_merge_down)), ctypes.byref(st),
        runs.ctypes.data if want_runs else None, nat.ctypes.data if want_runs else None,
        rows.ctypes.data if want_trace else None, cap, ctypes.byref(count),
    )
    _raise(code)
    stats = {f: int(getattr(st, f)) for f in STAT_FIELDS}
    r = stats["runs_detected"]
    res = OracleResult(keys, values, stats)
    if want_runs:
        res.run_lengths = runs[:r].tolist()
        res.natural_run_lengths = nat[:r].tolist()
    if want_trace:
        res.trace = trace_rows_to_list(rows[: count.value])
    return res


def detect_runs(keys, min_run_len=24):
    """The sort's run chain (run_lengths, natural_run_lengths) without sorting
    (policy.py:241-248 over runs.py:23-82); O(n), no copy of the input."""
    lib = _load()
    keys = np.ascontiguousarray(keys)
    if keys.dtype not in DTYPE_IDS:
        raise ValueError("unsupported dtype %s" % keys.dtype)
    n = keys.shape[0]
    r = lib.pso_detect_runs(DTYPE_IDS[keys.dtype], keys.ctypes.data, n, min_run_len, None, None, 0)
    if r < 0:
        _raise(-r)
    runs = np.zeros(max(r, 1), dtype=np.int64)
    nat = np.zeros(max(r, 1), dtype=np.int64)
    r2 = lib.pso_detect_runs(DTYPE_IDS[keys.dtype], keys.ctypes.data, n, min_run_len, runs.ctypes.data,
                             nat.ctypes.data, r)
    assert r2 == r
    return runs[:r], nat[:r]


def merge_cost_for_profile(lengths, k, strict_merge_down=False, want_trace=True):
    """policy.merge_cost_for_profile restated; returns (cost, trace, max_stack_height)."""
    lib = _load()
    lengths = np.ascontiguousarray(np.asarray(lengths, dtype=np.int64))
    r = lengths.shape[0]
    cap = max(r, 1) if want_trace else 0
    rows = np.zeros((cap, 7), dtype=np.int64) if want_trace else None
    cost = ctypes.c_int64(0)
    msh = ctypes.c_int64(0)
    count = ctypes.c_int64(0)
    code = lib.pso_merge_cost_for_profile(
        lengths.ctypes.data if r else None, r, k, int(bool(strict_merge_down)), ctypes.byref(cost),
        ctypes.byref(msh), rows.ctypes.data if want_trace else None, cap, ctypes.byref(count),
    )
    _raise(code)
    trace = trace_rows_to_list(rows[: count.value]) if want_trace else []
    return int(cost.value), trace, int(msh.value)


def node_power(k, n, b1, e1, b2, e2, any_k=False):
    v = _load().pso_node_power(k, n, b1, e1, b2, e2, int(bool(any_k)))
    if v < 0:
        _raise(-v)
    return v


def run_stack_capacity(k, n):
    v = _load().pso_run_stack_capacity(k, n)
    if v < 0:
        _raise(-v)
    return v


def stable_argsort_certificate(keys_in, keys_out, perm):
    """O(n) output certificate: keys_out == keys_in[perm]; perm is
    a permutation; keys nondecreasing under IEEE <=; equal keys keep
    increasing original index.  Returns None if OK else a message."""
    keys_in = np.asarray(keys_in)
    keys_out = np.asarray(keys_out)
    perm = np.asarray(perm).astype(np.int64)
    n = keys_in.shape[0]
    if keys_out.shape[0] != n or perm.shape[0] != n:
        return "length mismatch"
    if n == 0:
        return None
    seen = np.zeros(n, dtype=bool)
    if perm.min() < 0 or perm.max() >= n:
        return "perm out of range"
    seen[perm] = True
    if not seen.all():
        return "perm is not a permutation"
    if not np.array_equal(keys_in[perm].view(np.uint8), keys_out.view(np.uint8)):
        return "keys_out != keys_in[perm]"
    a, b = keys_out[:-1], keys_out[1:]
    if not np.all(a <= b):
        return "keys not sorted"
    eq = a == b
    if np.any(perm[:-1][eq] > perm[1:][eq]):
        return "equal keys out of input order"
    return None
