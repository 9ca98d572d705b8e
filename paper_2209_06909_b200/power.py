"""Boundary powers (mirrors power.py:24-96 of the reference).

``node_power`` and ``run_stack_capacity`` are evaluated by the C ABI
(``ps_node_power``, ``ps_run_stack_capacity``: exact 128-bit integer
arithmetic); the sort itself computes every power on the device with the
equivalent clz formula (csrc/ps_tree.cuh).
"""

from __future__ import annotations

from . import _lib


def ceil_log(k: int, n: int) -> int:
    """Smallest m >= 0 with k**m >= n (power.py:24-34)."""
    if k < 2:
        raise ValueError("ceil_log needs k >= 2")
    if n < 1:
        raise ValueError("ceil_log needs n >= 1")
    m, p = 0, 1
    while p < n:
        p *= k
        m += 1
    return m


def run_stack_capacity(k: int, n: int) -> int:
    """``(k-1) * (ceil(log_k n) + 1)`` (power.py:37-44)."""
    v = _lib.load().ps_run_stack_capacity(k, n)
    if v < 0:
        raise ValueError("run_stack_capacity needs k >= 2 and n >= 1")
    return v


def node_power(k: int, n: int, b1: int, e1: int, b2: int, e2: int) -> int:
    """Power of the boundary between runs [b1, e1) and [b2, e2) (power.py:47-55)."""
    v = _lib.load().ps_node_power(k, n, b1, e1, b2, e2, 0)
    if v < 0:
        _lib.check(-v)
    return v


def _node_power_any(k: int, n: int, b1: int, e1: int, b2: int, e2: int) -> int:
    v = _lib.load().ps_node_power(k, n, b1, e1, b2, e2, 1)
    if v < 0:
        _lib.check(-v)
    return v


def boundary_powers(lengths, k: int) -> list:
    """Powers of all r-1 interior boundaries of a profile (power.py:77-96)."""
    if not lengths:
        raise ValueError("a run profile has at least one run")
    if any(length < 1 for length in lengths):
        raise ValueError("run lengths must be positive")
    n = sum(lengths)
    out = []
    left = 0
    for j in range(len(lengths) - 1):
        mid = left + lengths[j]
        right = mid + lengths[j + 1]
        out.append(_node_power_any(k, n, left, mid, mid, right))
        left = mid
    return out
