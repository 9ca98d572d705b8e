"""SortStats and the analytic counters (mirrors statskit.py:75-124 of the
reference).

Every counter is exact: merge_cost, buffer_cost, max_stack_height,
runs_detected, merges2/3/4, scan_reads, scan_writes, run_lengths and
natural_run_lengths come from the merge tree; ``comparisons`` and ``moves``
(the reference's CountingOrder and element writes, statskit.py:49-72) from
closed forms over a few ranks per merge computed on the device.
They are ``None`` only when a sort was asked not to count them
(``SortConfig(count_comparisons=False)``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional


@dataclass(slots=True)
class SortStats:
    """Counters for one sort call (statskit.py:75-98)."""

    comparisons: Optional[int] = 0
    merge_cost: int = 0
    buffer_cost: int = 0
    moves: Optional[int] = 0
    max_stack_height: int = 0
    runs_detected: int = 0
    merges2: int = 0
    merges3: int = 0
    merges4: int = 0
    scan_reads: int = 0
    scan_writes: int = 0
    run_lengths: list = field(default_factory=list)
    natural_run_lengths: list = field(default_factory=list)
    # device of an asynchronous counting sort whose comparisons / moves are
    # still on the device (policy.finish_counters); not a reference field
    _pending: object = field(default=None, repr=False, compare=False)

    @property
    def merges_total(self) -> int:
        return self.merges2 + self.merges3 + self.merges4


def scanned_elements_estimate(stats: SortStats, n: int) -> int:
    """``4 * merge_cost + 2 * n`` (statskit.py:101-108)."""
    return 4 * stats.merge_cost + 2 * n


def normalized_merge_cost(value: float, n: int, min_run_len: int) -> float:
    """``value / (n * lg(n / min_run_len))`` (statskit.py:111-116)."""
    if n <= min_run_len:
        raise ValueError("normalization needs n > min_run_len")
    return value / (n * math.log2(n / min_run_len))


def normalized_time(milliseconds: float, n: int) -> float:
    """``ms * 1e6 / (n * lg n)`` (statskit.py:119-124)."""
    if n < 2:
        raise ValueError("normalization needs n >= 2")
    return milliseconds * 1e6 / (n * math.log2(n))
