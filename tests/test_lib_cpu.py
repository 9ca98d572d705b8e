"""CPU-side checks of the product library (no GPU needed): it builds, loads,
exports every symbol include/powersort_b200.h declares, and its host-side
helpers (node_power, run_stack_capacity, config validation) match the
reference's golden values."""

import ctypes
import os
import re

import pytest

import __graft_entry__ as ge
from paper_2209_06909_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    ge.build_lib()
    return _lib.load()


def test_header_symbols_are_exported(lib):
    header = open(os.path.join(REPO, "include", "powersort_b200.h")).read()
    declared = set(re.findall(r"\b(ps_[a-z_]+)\s*\(", header))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_node_power_matches_reference(lib, golden_powers):
    for k, n, b1, e1, b2, e2, p in golden_powers["powers"]:
        assert lib.ps_node_power(k, n, b1, e1, b2, e2, 1) == p
    for k, n, cap in golden_powers["caps"]:
        assert lib.ps_run_stack_capacity(k, n) == cap
    assert lib.ps_node_power(5, 4, 0, 2, 2, 4, 0) < 0
    assert lib.ps_node_power(2, 4, 0, 2, 3, 4, 0) < 0


def test_python_power_api(lib):
    from paper_2209_06909_b200 import node_power, run_stack_capacity
    from paper_2209_06909_b200.power import boundary_powers

    assert node_power(2, 4, 0, 2, 2, 4) == 1
    assert boundary_powers([2, 2, 4, 8], 2) == [3, 2, 1]
    assert boundary_powers([2, 2, 4, 8], 4) == [2, 1, 1]
    assert boundary_powers([4, 4, 4, 4, 48], 4) == [2, 2, 2, 1]
    assert run_stack_capacity(4, 10**6) == 33
    with pytest.raises(ValueError):
        node_power(5, 4, 0, 2, 2, 4)


def test_config_validation_without_gpu(lib):
    st = _lib.PsStats()
    for k, variant, mrl in ((3, 3, 24), (2, 3, 24), (4, 9, 24), (4, 3, 0)):
        cfg = _lib.PsConfig(k, variant, mrl, 0, 1)
        assert lib.ps_sort(0, None, None, 0, cfg, None, 0, st, None) == _lib.PS_EINVAL
    cfg = _lib.PsConfig(4, 3, 24, 0, 1)
    assert lib.ps_sort(0, None, None, 0, cfg, None, 0, st, None) == _lib.PS_OK  # n == 0
    assert lib.ps_workspace_size(1 << 20, 0, cfg) > (1 << 20) * 8


def test_shim_config_errors():
    from paper_2209_06909_b200 import SortConfig, stable_sort_with

    with pytest.raises(ValueError):
        stable_sort_with([1], SortConfig(k=3, variant="4way"))
    with pytest.raises(ValueError):
        stable_sort_with([1], SortConfig(k=2, variant="4way"))
    with pytest.raises(ValueError):
        stable_sort_with([1], SortConfig(k=4, variant="no-such-kernel"))
    with pytest.raises(ValueError):
        stable_sort_with([1], SortConfig(min_run_len=0))
