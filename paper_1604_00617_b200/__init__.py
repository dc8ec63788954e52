"""B200-native Accelerated Cyclic Reduction (arXiv 1604.00617) hot path.

Drop-in for the reference package's solve entry point
(``acrsolve.acr_solve``) and its input / parameter types.  The arithmetic
runs in hand-written sm_100a CUDA kernels behind the C ABI in
``include/acr_b200.h``; see DESIGN.md.
"""

from .problems import CONFIGS, make_config, random_system
from .system import (BlockTridiagSystem, RankProfile, SingularBlockError,
                     SolveReport, Tolerance)
from .tree import NodeTable, build_node_table

__version__ = "0.1.0"

__all__ = [
    "BlockTridiagSystem", "Tolerance", "SingularBlockError", "RankProfile",
    "SolveReport", "NodeTable", "build_node_table", "CONFIGS", "make_config",
    "random_system", "acr_solve", "AcrSolver", "expected_levels",
    "relative_residual_gpu",
]


def __getattr__(name):
    # the solver pulls in torch + the CUDA library lazily
    if name in ("acr_solve", "AcrSolver", "expected_levels",
                "relative_residual_gpu"):
        from . import solver
        return getattr(solver, name)
    raise AttributeError(name)
