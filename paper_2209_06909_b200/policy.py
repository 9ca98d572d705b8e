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
    #: B200 extension: compute the exact ``comparisons`` / ``moves`` counters of
    #: the reference's CountingOrder (statskit.py:49-72); the sort then waits
    #: for its merges.  Off: both are reported as None.
    count_comparisons: bool = False


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
    """Per-device workspace cache (grown on demand, torch caching allocator)."""

    def __init__(self):
        self.buf = {}
        self.stream = {}

    def get(self, device, nbytes):
        """The device's workspace for use on its current stream.  A sort returns
        with its merges still queued, so a switch of streams first orders the
        new stream after the last one, and a grown buffer replaces the old one
        only once the old one's work is done."""
        torch = _torch()
        cur = self.buf.get(device)
        stream = torch.cuda.current_stream(device)
        last = self.stream.get(device)
        if last is not None and last != stream:
            stream.wait_stream(last)
        if cur is None or cur.numel() < nbytes:
            if last is not None:
                last.synchronize()
            cur = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
            self.buf[device] = cur
        self.stream[device] = stream
        return cur


_WS = _Workspace()


def check(device=None):
    """Waits for the last sort on ``device`` (its merges run asynchronously)
    and raises if a device invariant was violated during them (ps_check)."""
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ws = _WS.buf.get(dev)
    if ws is None:
        return
    lib = _lib.load()
    _lib.check(lib.ps_check(ws.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))


def _cfg_struct(config, values_mode):
    return _lib.PsConfig(
        config.k, _lib.VARIANT_IDS[config.variant], config.min_run_len, int(bool(config.strict_merge_down)),
        values_mode, int(bool(getattr(config, "count_comparisons", False))), 0,
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
        ws = _WS.buf[torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())]
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


def _sort_tensor(keys, values, config, values_mode, collect_runs=True):
    """Core call: sorts ``keys`` (CUDA tensor) in place; ``values`` int32
    CUDA tensor permuted alongside (PERMUTE) or filled with source indices
    (ARGSORT).  Returns SortStats."""
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
    cfg = _cfg_struct(config, values_mode)
    if keys.data_ptr() % 16 or values.data_ptr() % 16:
        # the C ABI needs 16-byte aligned arrays (TMA); sort aligned copies of views
        k2, v2 = keys.clone(), values.clone()
        stats = _sort_tensor(k2, v2, config, values_mode, collect_runs)
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
    stats.comparisons = int(st.comparisons) if st.comparisons_valid else None
    stats.moves = int(st.moves) if st.moves_valid else None
    if collect_runs:
        stats.run_lengths, stats.natural_run_lengths = _read_runs(lib, ws, stats.runs_detected)
    if config.on_merge is not None:
        for entry in read_trace(ws):
            config.on_merge(entry)
    return stats


def stable_argsort(keys, config=None, collect_runs=True):
    """Sort the CUDA tensor ``keys`` in place; return ``(keys, perm, stats)``
    where ``perm`` (int32) holds the source index of every output element --
    the reference's (key, index) records after the sort."""
    torch = _torch()
    if config is None:
        config = SortConfig()
    perm = torch.empty(keys.numel(), dtype=torch.int32, device=keys.device)
    stats = _sort_tensor(keys, perm, config, _lib.VALUES_ARGSORT, collect_runs)
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


def _sort_list(lst, config):
    torch = _torch()
    n = len(lst)
    if n == 0:
        return SortStats()
    keyf = config.key
    ks = [keyf(x) for x in lst] if keyf is not None else list(lst)
    if all(isinstance(x, (int, np.integer)) and not isinstance(x, bool) for x in ks):
        arr = np.asarray(ks, dtype=np.int64)
    elif all(isinstance(x, (int, float, np.integer, np.floating)) for x in ks):
        arr = np.asarray(ks, dtype=np.float64)
    else:
        raise ValueError("list keys must be numbers")
    dev = torch.device("cuda", torch.cuda.current_device())
    keys = torch.from_numpy(arr).to(dev)
    plain = SortConfig(config.k, config.variant, config.min_run_len, None, config.strict_merge_down,
                       config.on_merge)
    _, perm, stats = stable_argsort(keys, plain)
    order = perm.cpu().numpy()
    lst[:] = [lst[i] for i in order.tolist()]
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
