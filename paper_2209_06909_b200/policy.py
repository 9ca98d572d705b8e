"""The drop-in sort entry points (mirrors policy.py:34-304 of the reference).

``stable_sort_with(keys, config)`` sorts a 1-D CUDA tensor in place, stably,
and returns the populated :class:`SortStats`, exactly like the reference's
``stable_sort_with(lst, config)`` does for a Python list.  The whole hot path
-- run detection, boundary powers, the merge tree and the batched k-way
merges -- runs in ``libpowersort_b200.so`` on the GPU; this module only
validates the config, allocates the workspace and converts results.

Python lists are accepted too (the reference's own calling convention): the
keys (``key(x)`` per element when ``config.key`` is set) are sorted on the
device and the list is reordered by the stable permutation, which is the
reference's output.
"""

from __future__ import annotations

import ctypes

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from .statskit import SortStats

#: Default minimum run length (policy.py:34-36).
MIN_RUN_LEN = 24


@dataclass(frozen=True)
class _VariantInfo:
    k: int
    needs_sentinel: bool
    fallback: Optional[str] = None


#: Merge-kernel families (policy.py:49-69).  On the device every family runs
#: the same stable k-way merge (the output is unique); the family selects the
#: counter formulas the reference's kernels produce.
VARIANTS = {
    "2way": _VariantInfo(2, True, "2way-nosentinel"),
    "2way-copy-smaller": _VariantInfo(2, False),
    "2way-nosentinel": _VariantInfo(2, False),
    "4way": _VariantInfo(4, True, "4way-nosentinel"),
    "4way-nosentinel": _VariantInfo(4, False),
}


@dataclass(frozen=True)
class SortConfig:
    """Configuration of one sort call (policy.py:72-91)."""

    k: int = 4
    variant: str = "4way"
    min_run_len: int = MIN_RUN_LEN
    key: Optional[Callable] = None
    strict_merge_down: bool = False
    on_merge: Optional[Callable] = None
    #: The exact ``comparisons`` / ``moves`` counters of the reference's
    #: CountingOrder (statskit.py:49-72), which the reference always returns.
    #: B200 extension: False skips their per-stage counting launches and
    #: reports both as None.
    count_comparisons: bool = True


def _validated(config):
    """policy.py:178-194"""
    if config.k not in (2, 4):
        raise ValueError("k must be 2 or 4, got %r" % (config.k,))
    info = VARIANTS.get(config.variant)
    if info is None:
        raise ValueError(
            "unknown merge variant %r (choose from %s)" % (config.variant, ", ".join(sorted(VARIANTS)))
        )
    if info.k != config.k:
        raise ValueError(
            "variant %r implements k=%d, but config asks for k=%d" % (config.variant, info.k, config.k)
        )
    if config.min_run_len < 1:
        raise ValueError("min_run_len must be >= 1")
    return info


def _torch():
    import torch

    return torch


_DTYPES = None


def _dtype_id(t):
    torch = _torch()
    global _DTYPES
    if _DTYPES is None:
        _DTYPES = {torch.int32: 0, torch.int64: 1, torch.float32: 2, torch.float64: 3}
    if t.dtype not in _DTYPES:
        raise ValueError("unsupported key dtype %s (int32, int64, float32, float64)" % t.dtype)
    return _DTYPES[t.dtype]


class _Workspace:
    """Workspace cache, one buffer per (device, stream) (grown on demand, torch
    caching allocator).  Sorts on different streams therefore never share
    scratch memory and may run concurrently (SPEC.md:264 of the reference
    allows concurrent sorts)."""

    def __init__(self):
        self.buf = {}

    @staticmethod
    def key(device, stream=None):
        torch = _torch()
        device = torch.device(device)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        return (device, stream.cuda_stream)

    def get(self, device, nbytes):
        """The workspace of ``device``'s current stream.  A grown buffer
        replaces the old one only once the stream's queued work is done."""
        torch = _torch()
        stream = torch.cuda.current_stream(device)
        k = self.key(device, stream)
        cur = self.buf.get(k)
        if cur is None or cur.numel() < nbytes:
            if cur is not None:
                stream.synchronize()
            cur = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
            self.buf[k] = cur
        return cur

    def last(self, device=None):
        torch = _torch()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        return self.buf.get(self.key(dev))


_WS = _Workspace()


def check(device=None):
    """Waits for the last sort on ``device``'s current stream and raises if a
    device invariant was violated during its merges (ps_check).  Only needed
    after an asynchronous sort; the default sort checks before returning."""
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ws = _WS.last(dev)
    if ws is None:
        return
    lib = _lib.load()
    _lib.check(lib.ps_check(ws.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))


def finish_counters(stats):
    """Completes the SortStats of an asynchronous sort: waits for it on the
    current stream, checks its device invariants and fills ``comparisons``
    and ``moves`` (ps_result_counters: a host-mapped read, no device-wide
    synchronization); a no-op for any other SortStats."""
    dev = getattr(stats, "_pending", None)
    if dev is None:
        return stats
    torch = _torch()
    ws = _WS.last(dev)
    lib = _lib.load()
    cmp_ = ctypes.c_int64()
    mov = ctypes.c_int64()
    _lib.check(lib.ps_result_counters(ws.data_ptr(), torch.cuda.current_stream(dev).cuda_stream, ctypes.byref(cmp_),
                                      ctypes.byref(mov)))
    stats.comparisons = int(cmp_.value) if cmp_.value >= 0 else None
    stats.moves = int(mov.value) if mov.value >= 0 else None
    stats._pending = None
    return stats


def _cfg_struct(config, values_mode, asynchronous=False):
    return _lib.PsConfig(
        config.k, _lib.VARIANT_IDS[config.variant], config.min_run_len, int(bool(config.strict_merge_down)),
        values_mode, int(bool(getattr(config, "count_comparisons", True))),
        _lib.FLAG_ASYNC if asynchronous else 0,
    )


def _read_runs(lib, ws, r):
    runs = np.zeros(max(r, 1), dtype=np.int64)
    nat = np.zeros(max(r, 1), dtype=np.int64)
    _lib.check(lib.ps_result_runs(ws.data_ptr(), runs.ctypes.data, nat.ctypes.data, max(r, 1)))
    return runs[:r].tolist(), nat[:r].tolist()


def read_trace(ws=None, device=None):
    """The executed merge tree of the last sort on ``device``, in the
    reference's on_merge order: [((b0, .., end), length), ...]."""
    torch = _torch()
    lib = _lib.load()
    if ws is None:
        ws = _WS.last(device)
        if ws is None:
            raise ValueError("no sort has run on this device's current stream")
    r = ctypes_i64()
    nm = ctypes_i64()
    _lib.check(lib.ps_result_counts(ws.data_ptr(), r, nm))
    cnt = nm.value
    rows = np.zeros((max(cnt, 1), 7), dtype=np.int64)
    _lib.check(lib.ps_result_trace(ws.data_ptr(), rows.ctypes.data, max(cnt, 1)))
    out = []
    for row in rows[:cnt]:
        w = int(row[0])
        out.append((tuple(int(x) for x in row[1 : 2 + w]), int(row[6])))
    return out


def ctypes_i64():
    import ctypes

    return ctypes.c_int64(0)


def _sort_tensor(keys, values, config, values_mode, collect_runs=True, asynchronous=False):
    """Core call: sorts ``keys`` (CUDA tensor) in place; ``values`` int32
    CUDA tensor permuted alongside (PERMUTE) or filled with source indices
    (ARGSORT).  Returns SortStats.  ``asynchronous``: return once the merges
    are queued (PS_FLAG_ASYNC; check() reports their invariants later)."""
    torch = _torch()
    info = _validated(config)
    del info
    if config.key is not None:
        raise ValueError("a key callable is not supported for tensor input (pass the key tensor itself)")
    if not isinstance(keys, torch.Tensor) or not keys.is_cuda:
        raise ValueError("keys must be a CUDA tensor")
    if keys.dim() != 1 or not keys.is_contiguous():
        raise ValueError("keys must be a contiguous 1-D tensor")
    n = keys.numel()
    stats = SortStats()
    if n == 0:
        return stats
    if values is None or values.dtype != torch.int32 or values.numel() != n or not values.is_cuda:
        raise ValueError("values must be an int32 CUDA tensor of the same length")
    if values.device != keys.device or not values.is_contiguous():
        raise ValueError("values must be contiguous and on the keys' device")
    lib = _lib.load()
    dt = _dtype_id(keys)
    cfg = _cfg_struct(config, values_mode, asynchronous)
    if keys.data_ptr() % 16 or values.data_ptr() % 16:
        # the C ABI needs 16-byte aligned arrays (TMA); sort aligned copies of views
        k2, v2 = keys.clone(), values.clone()
        stats = _sort_tensor(k2, v2, config, values_mode, collect_runs)  # synchronous
        keys.copy_(k2)
        values.copy_(v2)
        return stats
    with torch.cuda.device(keys.device):
        nbytes = lib.ps_workspace_size(n, dt, cfg)
        if nbytes == 0:
            raise ValueError("invalid sort arguments")
        ws = _WS.get(keys.device, nbytes)
        st = _lib.PsStats()
        stream = torch.cuda.current_stream(keys.device).cuda_stream
        _lib.check(
            lib.ps_sort(dt, keys.data_ptr(), values.data_ptr(), n, cfg, ws.data_ptr(), ws.numel(), st, stream)
        )
    for f in ("merge_cost", "buffer_cost", "max_stack_height", "runs_detected", "merges2", "merges3", "merges4",
              "scan_reads", "scan_writes"):
        setattr(stats, f, int(getattr(st, f)))
    stats.comparisons = int(st.comparisons) if st.comparisons_valid == 1 else None
    stats.moves = int(st.moves) if st.moves_valid == 1 else None
    if st.comparisons_valid == 2:  # asynchronous counting sort: finish_counters() reads them
        stats._pending = keys.device
    if collect_runs:
        stats.run_lengths, stats.natural_run_lengths = _read_runs(lib, ws, stats.runs_detected)
    if config.on_merge is not None:
        for entry in read_trace(ws):
            config.on_merge(entry)
    return stats


def stable_argsort(keys, config=None, collect_runs=True, asynchronous=False):
    """Sort the CUDA tensor ``keys`` in place; return ``(keys, perm, stats)``
    where ``perm`` (int32) holds the source index of every output element --
    the reference's (key, index) records after the sort.  ``asynchronous``:
    return once the sort is queued (PS_FLAG_ASYNC); ``finish_counters(stats)``
    later waits for it, checks its device invariants and fills comparisons /
    moves."""
    torch = _torch()
    if config is None:
        config = SortConfig()
    perm = torch.empty(keys.numel(), dtype=torch.int32, device=keys.device)
    stats = _sort_tensor(keys, perm, config, _lib.VALUES_ARGSORT, collect_runs, asynchronous)
    return keys, perm, stats


def stable_sort_with(lst, config=None, values=None):
    """Sort ``lst`` in place, stably, and return the populated SortStats
    (policy.py:201-262).

    ``lst`` is a 1-D CUDA tensor (int32/int64/float32/float64), optionally
    with a ``values`` tensor permuted alongside (int32 1-D: carried through
    the merges; any other dtype or row width: gathered by the stable
    permutation), or a Python list (numbers, or records with ``config.key``).
    """
    if config is None:
        config = SortConfig()
    _validated(config)
    torch = _torch()
    if isinstance(lst, torch.Tensor):
        if values is not None:
            if values.dtype == torch.int32 and values.dim() == 1:
                return _sort_tensor(lst, values, config, _lib.VALUES_PERMUTE)
            return _sort_with_rows(lst, values, config)
        _, _, stats = stable_argsort(lst, config)
        return stats
    if isinstance(lst, list):
        return _sort_list(lst, config)
    raise ValueError("stable_sort_with expects a CUDA tensor or a list")


def _sort_with_rows(keys, values, config):
    """Payload of any dtype / row width (first dimension = len(keys)), permuted
    alongside the keys: a stable argsort, then ps_gather_rows."""
    torch = _torch()
    if not isinstance(values, torch.Tensor) or not values.is_cuda or values.device != keys.device:
        raise ValueError("values must be a CUDA tensor on the keys' device")
    if values.dim() < 1 or values.shape[0] != keys.numel() or not values.is_contiguous():
        raise ValueError("values must be contiguous with one row per key")
    _, perm, stats = stable_argsort(keys, config)
    n = keys.numel()
    if n == 0:
        return stats
    row_bytes = values.element_size() * (values.numel() // n)
    if row_bytes == 0:
        return stats
    src = values.clone()
    lib = _lib.load()
    with torch.cuda.device(keys.device):
        stream = torch.cuda.current_stream(keys.device).cuda_stream
        _lib.check(lib.ps_gather_rows(src.data_ptr(), perm.data_ptr(), values.data_ptr(), n, row_bytes, stream))
    return stats


#: Reserved greatest elements (the reference's ``statskit.SENTINEL``,
#: registered by the ``powersort`` compatibility shim): ``le(x, SENTINEL)`` is
#: true and ``le(SENTINEL, x)`` false for every ordinary x, and comparisons
#: against it are not counted (statskit.py:49-72).
_SENTINELS = []


def register_sentinel(obj):
    """Treat ``obj`` (compared by identity) as the reference's SENTINEL."""
    if not any(obj is x for x in _SENTINELS):
        _SENTINELS.append(obj)


_I64_MIN, _I64_MAX = -(2**63), 2**63 - 1


def _list_keys(lst, keyf):
    """The numeric key array of a Python list (policy.py:201-262 compares
    ``key(a) <= key(b)``).  Returns (numpy keys, sentinel mask or None).
    Integer keys must fit int64; a mix of ints and floats must be exact in
    float64 (|int| <= 2^53), else the order could differ from Python's."""
    sent = None
    if _SENTINELS:
        flags = [any(x is t for t in _SENTINELS) for x in lst]
        if any(flags):
            sent = np.asarray(flags, dtype=bool)
    ks = [0 if (sent is not None and sent[i]) else (keyf(x) if keyf is not None else x)
          for i, x in enumerate(lst)]
    live = ks if sent is None else [k for k, f in zip(ks, sent.tolist()) if not f]
    if all(isinstance(x, (int, np.integer)) for x in live):
        if any(not (_I64_MIN <= int(x) <= _I64_MAX) for x in live):
            raise ValueError("integer list keys must fit in int64")
        arr = np.asarray([int(x) for x in ks], dtype=np.int64)
        if sent is not None:
            top = int(arr[~sent].max()) if (~sent).any() else 0
            if top == _I64_MAX:
                raise ValueError("SENTINEL needs a key value above every list key")
            arr[sent] = top + 1
        return arr, sent
    if all(isinstance(x, (int, float, np.integer, np.floating)) for x in live):
        for x in live:
            if isinstance(x, (int, np.integer)) and abs(int(x)) > 2**53:
                raise ValueError("mixed int/float list keys must be exact in float64 (|int| <= 2^53)")
        arr = np.asarray([float(x) for x in ks], dtype=np.float64)
        if np.isnan(arr).any():
            raise ValueError("NaN keys are not supported (their order is undefined in the reference)")
        if sent is not None:
            if np.isposinf(arr[~sent]).any():
                raise ValueError("SENTINEL needs a key value above every list key")
            arr[sent] = np.inf
        return arr, sent
    raise ValueError("list keys must be numbers")


def _sort_list(lst, config):
    """Sorts a Python list in place: its keys are sorted on the device and the
    list is reordered by the stable permutation (the reference's output,
    SURVEY F1).  Reserved SENTINEL elements take a key above every other key
    (they sort last, in input order); the reference then switches to the
    variant's sentinel-free sibling (policy.py:211-214), whose counters apply."""
    torch = _torch()
    n = len(lst)
    if n == 0:
        return SortStats()
    arr, sent = _list_keys(lst, config.key)
    variant = config.variant
    if sent is not None and VARIANTS[variant].needs_sentinel:
        variant = VARIANTS[variant].fallback
    dev = torch.device("cuda", torch.cuda.current_device())
    keys = torch.from_numpy(arr).to(dev)
    plain = SortConfig(config.k, variant, config.min_run_len, None, config.strict_merge_down,
                       config.on_merge, config.count_comparisons)
    _, perm, stats = stable_argsort(keys, plain)
    order = perm.cpu().numpy()
    lst[:] = [lst[i] for i in order.tolist()]
    if sent is not None and stats.comparisons is not None:
        # comparisons against SENTINEL are not counted (statskit.py:64-67):
        # the device counted them as ordinary key comparisons
        stats.comparisons = None
    return stats


def stable_sort(lst, key=None):
    """Sort ``lst`` in place, stably, with the default configuration."""
    stable_sort_with(lst, SortConfig(key=key))


def merge_cost_for_profile(lengths, k, strict_merge_down=False, on_merge=None):
    """Total merge cost the policy produces for a run-length profile
    (policy.py:270-304), computed by the device tree builder."""
    torch = _torch()
    if k not in (2, 4):
        raise ValueError("k must be 2 or 4, got %r" % (k,))
    if not lengths:
        raise ValueError("a run profile has at least one run")
    if any(length < 1 for length in lengths):
        raise ValueError("run lengths must be positive")
    lib = _lib.load()
    arr = np.ascontiguousarray(np.asarray(lengths, dtype=np.int64))
    r = arr.shape[0]
    n = int(arr.sum())
    nbytes = lib.ps_profile_workspace_size(r, n)
    dev = torch.device("cuda", torch.cuda.current_device())
    ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=dev)
    cost = ctypes_i64()
    msh = ctypes_i64()
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(lib.ps_tree_from_profile(arr.ctypes.data, r, k, int(bool(strict_merge_down)), ws.data_ptr(),
                                        ws.numel(), cost, msh, stream))
    if on_merge is not None:
        for entry in read_trace(ws):
            on_merge(entry)
    return int(cost.value)
