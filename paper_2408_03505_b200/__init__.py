"""B200-native hot path of Optimus (arXiv 2408.03505): batched evaluation of the
bubble-scheduling search behind a C ABI (include/optimus.h), sm_100a kernels in
csrc/, and a thin ctypes binding (optimus.py)."""
from .optimus import (  # noqa: F401
    Ctx,
    OptimusError,
    Problem,
    optimus_load_costs,
    optimus_plan_only,
    optimus_workspace_bytes,
    search,
)
