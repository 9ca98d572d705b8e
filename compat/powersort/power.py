"""``powersort.power`` (power.py:24-96 of the reference) from the B200
package: exact powers through the C ABI (ps_node_power)."""

from paper_2209_06909_b200.power import (  # noqa: F401
    _node_power_any,
    boundary_powers,
    ceil_log,
    node_power,
    run_stack_capacity,
)
