"""``powersort`` compatibility shim over the B200 package.

Importing ``powersort`` with ``compat/`` first on ``sys.path`` gives the
reference package's public surface (``/root/reference/pkg/src/powersort/
__init__.py:9-47``) with the sort entry points -- ``stable_sort``,
``stable_sort_with``, ``merge_cost_for_profile``, ``SortConfig``,
``VARIANTS``, ``SortStats``, ``node_power``, ``run_stack_capacity``,
``scanned_elements_estimate`` -- served by ``paper_2209_06909_b200`` (the
CUDA path).  The remaining names (``MergeBuffer``, ``Run``, ``SENTINEL``,
``CountingOrder`` and the ``oracle`` / ``merges`` / ``runs`` / ``harness``
submodules) are the reference's own, loaded from its install under
``baseline/_ref``, so that the reference's test suite runs unmodified
against the GPU package (tests/test_reference_suite.py).
"""

from __future__ import annotations

import sys

from . import _ref

_r = _ref.load()
for _m in ("oracle", "merges", "runs", "harness"):
    sys.modules[__name__ + "." + _m] = _ref.sub(_m)

from . import policy, power, statskit  # noqa: E402
from .policy import (  # noqa: E402
    MIN_RUN_LEN,
    VARIANTS,
    SortConfig,
    merge_cost_for_profile,
    stable_sort,
    stable_sort_with,
)
from .power import node_power, run_stack_capacity  # noqa: E402
from .statskit import (  # noqa: E402
    SENTINEL,
    CountingOrder,
    SortStats,
    normalized_merge_cost,
    normalized_time,
    scanned_elements_estimate,
)

MergeBuffer = _r.MergeBuffer
Run = _r.Run
oracle = sys.modules[__name__ + ".oracle"]
merges = sys.modules[__name__ + ".merges"]
runs = sys.modules[__name__ + ".runs"]
harness = sys.modules[__name__ + ".harness"]

__version__ = "0.1.0"

__all__ = [
    "MIN_RUN_LEN",
    "MergeBuffer",
    "Run",
    "SENTINEL",
    "CountingOrder",
    "SortConfig",
    "SortStats",
    "VARIANTS",
    "merge_cost_for_profile",
    "node_power",
    "normalized_merge_cost",
    "normalized_time",
    "run_stack_capacity",
    "scanned_elements_estimate",
    "stable_sort",
    "stable_sort_with",
]
