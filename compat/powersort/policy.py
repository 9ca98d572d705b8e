"""``powersort.policy``: the sort entry points of the B200 package
(policy.py:34-304 of the reference); the stack machinery (``RunStack``,
``_merge_one_group``, ``_merge_down``) is the reference's, for its own tests."""

from paper_2209_06909_b200.policy import (  # noqa: F401
    MIN_RUN_LEN,
    VARIANTS,
    SortConfig,
    _validated,
    merge_cost_for_profile,
    stable_sort,
    stable_sort_with,
)

from . import _ref

_p = _ref.sub("policy")
RunStack = _p.RunStack
_merge_one_group = _p._merge_one_group
_merge_down = _p._merge_down
_contains_sentinel = _p._contains_sentinel
