"""Loads the reference package (the unmodified ``powersort`` installed under
``baseline/_ref`` by ``pip install --target``) under the private name
``_powersort_ref``, for the parts of its surface that are not the sort:
the analysis oracle, the CPU merge kernels, run detection helpers, RunStack,
CountingOrder / SENTINEL and the harness.  Test infrastructure of the shim
only; the sort itself never runs through it."""

from __future__ import annotations

import importlib.util
import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAME = "_powersort_ref"


def location():
    base = os.environ.get("PS_REFERENCE_PKG") or os.path.join(_REPO, "baseline", "_ref")
    return os.path.join(base, "powersort")


def load():
    """The reference package module (imported once)."""
    if NAME in sys.modules:
        return sys.modules[NAME]
    path = location()
    init = os.path.join(path, "__init__.py")
    if not os.path.exists(init):
        raise ImportError("the reference package is not installed at %s (see tools/stage_reference.sh)" % path)
    spec = importlib.util.spec_from_file_location(NAME, init, submodule_search_locations=[path])
    mod = importlib.util.module_from_spec(spec)
    sys.modules[NAME] = mod
    spec.loader.exec_module(mod)
    return mod


def sub(name):
    load()
    return importlib.import_module(NAME + "." + name)
