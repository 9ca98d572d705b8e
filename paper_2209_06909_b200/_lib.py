"""ctypes binding of ``libpowersort_b200.so`` (the C ABI in
``include/powersort_b200.h``).

There is no fallback: if the shared library is missing or no CUDA device is
usable, every sort raises.  Build it with ``python -c "import
__graft_entry__ as g; g.build()"`` (nvcc, sm_100a).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PS_LIB") or os.path.join(_HERE, "libpowersort_b200.so")

PS_OK, PS_EINVAL, PS_ECUDA, PS_ENOMEM, PS_EINVARIANT, PS_EOVERFLOW = range(6)

DTYPE_IDS = {"int32": 0, "int64": 1, "float32": 2, "float64": 3}
VARIANT_IDS = {"2way": 0, "2way-copy-smaller": 1, "2way-nosentinel": 2, "4way": 3, "4way-nosentinel": 4}
VALUES_PERMUTE, VALUES_ARGSORT = 0, 1
FLAG_ASYNC = 1

# Exported symbols (tests check the library exports every one of them).
EXPORTS = (
    "ps_workspace_size",
    "ps_sort",
    "ps_check",
    "ps_result_counts",
    "ps_result_counters",
    "ps_result_runs",
    "ps_result_trace",
    "ps_profile_workspace_size",
    "ps_tree_from_profile",
    "ps_node_power",
    "ps_run_stack_capacity",
    "ps_shard_merge_workspace_size",
    "ps_shard_merge",
    "ps_shard_sample_count",
    "ps_shard_samples",
    "ps_ipc_export",
    "ps_ipc_open",
    "ps_ipc_close",
    "ps_gather_rows",
    "ps_profile_enable",
    "ps_profile_read",
    "ps_launch_count",
    "ps_last_error",
    "ps_version",
)


class PsConfig(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int32),
        ("variant", ctypes.c_int32),
        ("min_run_len", ctypes.c_int64),
        ("strict_merge_down", ctypes.c_int32),
        ("values_mode", ctypes.c_int32),
        ("count_comparisons", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


class PsStats(ctypes.Structure):
    _fields_ = [
        ("comparisons", ctypes.c_int64),
        ("merge_cost", ctypes.c_int64),
        ("buffer_cost", ctypes.c_int64),
        ("moves", ctypes.c_int64),
        ("max_stack_height", ctypes.c_int64),
        ("runs_detected", ctypes.c_int64),
        ("merges2", ctypes.c_int64),
        ("merges3", ctypes.c_int64),
        ("merges4", ctypes.c_int64),
        ("scan_reads", ctypes.c_int64),
        ("scan_writes", ctypes.c_int64),
        ("comparisons_valid", ctypes.c_int32),
        ("moves_valid", ctypes.c_int32),
    ]


class PsProfEntry(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("stage", ctypes.c_int32),
        ("nodes", ctypes.c_int64),
        ("chunks", ctypes.c_int64),
        ("bytes", ctypes.c_int64),
        ("ms", ctypes.c_float),
        ("pad", ctypes.c_float),
    ]


PROF_KINDS = {0: "run_detection", 1: "merge_tree", 2: "leaf_formation", 3: "partition", 4: "merge"}

_lib = None


def load():
    """Load the library (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            "libpowersort_b200.so not found at %s -- build it with __graft_entry__.build() "
            "(the B200 path has no CPU fallback)" % LIB_PATH
        )
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    i64p = ctypes.POINTER(ctypes.c_int64)
    lib.ps_workspace_size.argtypes = [i64, i32, ctypes.POINTER(PsConfig)]
    lib.ps_workspace_size.restype = sz
    lib.ps_sort.argtypes = [i32, vp, vp, i64, ctypes.POINTER(PsConfig), vp, sz, ctypes.POINTER(PsStats), vp]
    lib.ps_check.argtypes = [vp, vp]
    lib.ps_sort.restype = ctypes.c_int
    lib.ps_result_counts.argtypes = [vp, i64p, i64p]
    lib.ps_result_counts.restype = ctypes.c_int
    lib.ps_result_runs.argtypes = [vp, vp, vp, i64]
    lib.ps_result_runs.restype = ctypes.c_int
    lib.ps_result_trace.argtypes = [vp, vp, i64]
    lib.ps_result_trace.restype = ctypes.c_int
    lib.ps_profile_workspace_size.argtypes = [i64, i64]
    lib.ps_profile_workspace_size.restype = sz
    lib.ps_tree_from_profile.argtypes = [vp, i64, i32, i32, vp, sz, i64p, i64p, vp]
    lib.ps_tree_from_profile.restype = ctypes.c_int
    lib.ps_node_power.argtypes = [i32, i64, i64, i64, i64, i64, i32]
    lib.ps_node_power.restype = ctypes.c_int
    lib.ps_run_stack_capacity.argtypes = [i64, i64]
    lib.ps_run_stack_capacity.restype = i64
    lib.ps_gather_rows.argtypes = [vp, vp, vp, i64, i64, vp]
    lib.ps_gather_rows.restype = i32
    lib.ps_shard_merge_workspace_size.argtypes = [i32, i64]
    lib.ps_shard_merge_workspace_size.restype = sz
    lib.ps_shard_merge.argtypes = [i32, i32, vp, vp, vp, vp, i64, i64, vp, vp, vp, sz, vp]
    lib.ps_shard_merge.restype = ctypes.c_int
    lib.ps_result_counters.argtypes = [vp, vp, vp, vp]
    lib.ps_result_counters.restype = ctypes.c_int
    lib.ps_shard_sample_count.argtypes = [i32, i64]
    lib.ps_shard_sample_count.restype = i64
    lib.ps_shard_samples.argtypes = [i32, vp, i64, vp, vp]
    lib.ps_ipc_export.argtypes = [i32, vp, vp, i64p]
    lib.ps_ipc_export.restype = ctypes.c_int
    lib.ps_ipc_open.argtypes = [i32, vp, ctypes.POINTER(ctypes.c_void_p)]
    lib.ps_ipc_open.restype = ctypes.c_int
    lib.ps_ipc_close.argtypes = [i32, vp]
    lib.ps_ipc_close.restype = ctypes.c_int
    lib.ps_shard_samples.restype = ctypes.c_int
    lib.ps_profile_enable.argtypes = [i32]
    lib.ps_profile_enable.restype = ctypes.c_int
    lib.ps_profile_read.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_int32)]
    lib.ps_profile_read.restype = ctypes.c_int
    lib.ps_launch_count.argtypes = []
    lib.ps_launch_count.restype = i64
    lib.ps_last_error.argtypes = []
    lib.ps_last_error.restype = ctypes.c_char_p
    lib.ps_version.argtypes = []
    lib.ps_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(code):
    """Map a ps_status to the reference's exception types (policy.py:178-194,
    :114-120, merges.py:63-72, power.py:53-66)."""
    if code == PS_OK:
        return
    msg = load().ps_last_error().decode(errors="replace")
    if code == PS_EINVAL:
        raise ValueError(msg)
    if code == PS_ENOMEM:
        raise MemoryError(msg)
    if code == PS_EINVARIANT:
        raise AssertionError(msg)
    if code == PS_EOVERFLOW:
        raise OverflowError(msg)
    raise RuntimeError(msg)


def profile_read():
    """Phase entries of the last profiled ps_sort on this thread."""
    lib = load()
    cnt = ctypes.c_int32(0)
    lib.ps_profile_read(None, 0, ctypes.byref(cnt))
    arr = (PsProfEntry * max(cnt.value, 1))()
    lib.ps_profile_read(arr, cnt.value, ctypes.byref(cnt))
    return [
        dict(kind=PROF_KINDS.get(e.kind, str(e.kind)), stage=e.stage, nodes=e.nodes, chunks=e.chunks,
             bytes=e.bytes, ms=e.ms)
        for e in arr[: cnt.value]
    ]
