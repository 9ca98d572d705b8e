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

# Names the reference's tests monkeypatch on this module (e.g.
# test_statskit.py:96 swaps SortStats to spy on the sort's stats object) are
# forwarded to the implementing module, so the patch reaches the sort.
import sys as _sys  # noqa: E402
import types as _types  # noqa: E402

from paper_2209_06909_b200 import policy as _impl  # noqa: E402

SortStats = _impl.SortStats


class _ForwardingModule(_types.ModuleType):
    _FORWARD = ("SortStats", "SortConfig", "VARIANTS", "MIN_RUN_LEN")

    def __setattr__(self, name, value):
        if name in self._FORWARD:
            setattr(_impl, name, value)
        super().__setattr__(name, value)


_sys.modules[__name__].__class__ = _ForwardingModule
