"""B200-native recycling Krylov solvers (arXiv:1501.03358): rGCROT(m,k),
rBiCGStab with one recycle space, GMRES(m)/BiCGStab (k = 0) and the hybrid
rGCROT -> rBiCGStab strategy, for sequences of structured-grid systems.

The solver is librk.so (hand-written CUDA for sm_100a behind the C-ABI of
include/rk.h); this package is its thin binding.  Importing it does not load
the library; the first call does, and fails loudly if it was not built."""
from ._lib import RkError, lib, EXPORTED, OUTCOME_NAMES
from .api import (Context, GridOperator, Solver, make_config, config_from_params,
                  solve_sequence, nccl_unique_id)

__all__ = ["RkError", "lib", "EXPORTED", "OUTCOME_NAMES", "Context", "GridOperator", "Solver",
           "make_config", "config_from_params", "solve_sequence", "nccl_unique_id"]
