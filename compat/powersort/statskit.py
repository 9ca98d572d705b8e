"""``powersort.statskit``: SortStats and the estimates from the B200 package;
``SENTINEL`` and ``CountingOrder`` are the reference's objects (statskit.py:
33-72), and SENTINEL is registered with the B200 list path so that lists
holding it sort it last (policy.py:211-214)."""

from paper_2209_06909_b200.policy import register_sentinel
from paper_2209_06909_b200.statskit import (  # noqa: F401
    SortStats,
    normalized_merge_cost,
    normalized_time,
    scanned_elements_estimate,
)

from . import _ref

_s = _ref.sub("statskit")
SENTINEL = _s.SENTINEL
CountingOrder = _s.CountingOrder
register_sentinel(SENTINEL)
