"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the SPFOM method: it only draws random
instances (consideration sets, attraction/shadow weights, prices, arrival
rates, capacities) and block-sampling sequences, following the BASELINE.json
config recipes.  Both `oracle/` and
`paper_2602_22421_b200/` consume its output; neither is imported here.
"""
from .generate import (  # noqa: F401
    CONFIGS,
    Instance,
    block_sequence,
    config_spec,
    generate,
    period_slice,
    stack_periods,
    with_bundles,
)
