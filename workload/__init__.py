"""Seeded synthetic workload generator (inputs only).

This module builds the integer-nanosecond cost tables that BOTH the CPU oracle
(`oracle/`) and the CUDA path (`paper_2408_03505_b200/`) consume.  It holds
none of the method's arithmetic (no pipeline simulation, no bubble packing, no
search): only the cost model that turns model shapes into per-kernel durations
 and counter-based random streams.
"""
from .gen import (  # noqa: F401
    CONFIGS,
    config_problem,
    toy_problem,
    random_problem,
    splitmix64,
    sample_indices,
    sample_indices_np,
    problem_summary,
)
