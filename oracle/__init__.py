"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct NumPy fp64 implementation of what the
B200 hot path computes (Alg. 1-4, eqs. (2)-(12)), written from
the paper in its order and notation.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl
reference` legs may import it.  The product package
`paper_1501_03358_b200` never imports it and shares no code with it; the
two meet only on the seeded inputs from `problems/`.

Pins (what ties each function to something other than itself) are listed
in each module header and in DESIGN.md "Oracle and pins".  The line-14a
recycle-space update (krylov.gcrot_update) is pinned by what one cycle
fixes -- every added column comes from the cycle's search space (the
post-cycle residual is orthogonal to all of C), u1 is parallel to the
cycle's correction, A_hat U = C, C^T C = I, T1 keeps the newest columns --
but the paper names the step without an algorithm, so which
second candidate p1 = 2 picks (argmax |y_j|, reading D11) is a choice no
passage can pin.
"""
from .stencil import Operator, shifted, to_dense, jacobi, Jacobi
from .krylov import (
    Report,
    refresh_space,
    gcrot_update,
    rgcrot,
    gmres,
    rbicgstab,
    bicgstab,
    run_sequence,
)

__all__ = [
    "Operator", "shifted", "to_dense", "jacobi", "Jacobi",
    "Report", "refresh_space", "gcrot_update", "rgcrot", "gmres",
    "rbicgstab", "bicgstab", "run_sequence",
]
