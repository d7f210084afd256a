"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the recycling method (no SpMV, no
preconditioner, no Krylov step).  It only manufactures the inputs the
paper's method consumes: banded (diagonal-storage) stencil coefficients
of a structured-grid operator A ("structured banded
sparse storage format ... 7 or 19 point stencil") and a sequence of
right-hand sides b_t.  Both `oracle/` and the
product binding / bench read these arrays; neither side imports the other.

The recipes are the synthetic stand-ins of BASELINE.json configs c1..c5
(the paper's GenIDLEST channel and porous-media systems are not
available); every reading is listed in DESIGN.md ("Input recipe").
"""
from .rng import splitmix64, uniform, uniform01
from .stencils import (
    OFFSETS7,
    OFFSETS19,
    StencilProblem,
    convection_diffusion_c1,
    channel19,
    porous7,
)
from .workloads import (
    SolverParams,
    Workload,
    WORKLOADS,
    get_workload,
    slab_range,
)

__all__ = [
    "splitmix64", "uniform", "uniform01",
    "OFFSETS7", "OFFSETS19", "StencilProblem",
    "convection_diffusion_c1", "channel19", "porous7",
    "SolverParams", "Workload", "WORKLOADS", "get_workload", "slab_range",
]
