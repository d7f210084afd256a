"""Small librk workload for compute-sanitizer runs (one tool per process):
the fused chain (forced), block Jacobi, SSOR, rGCROT/hybrid solves, T2."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RK_FORCE_CHAIN"] = "1"
import paper_1501_03358_b200 as rk  # noqa: E402
from problems import get_workload  # noqa: E402

ctx = rk.Context(0)
for name in ("c3m", "c2s"):
    w = get_workload(name)
    prob = w.problem()
    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets,
                         torch.from_numpy(prob.bands()).cuda(), prob.periodic)
    r = torch.from_numpy(prob.rhs(0).reshape(-1)).cuda()
    op.precond(r)
    op.precond(r, zblocks=2)
    op.precond(r, kind=2, omega_l=1.0)
    s = rk.Solver(op, rk.config_from_params(w.params))
    reps = rk.solve_sequence(s, lambda t: torch.from_numpy(prob.rhs(t).reshape(-1)).cuda(), 3,
                             w.params.method, n_sw=2)
    print(name, [r_["krylov_matvecs"] for r_ in reps], [r_["outcome"] for r_ in reps], flush=True)
    s.close()
    op.close()
torch.cuda.synchronize()
print("sanitize case ok")
