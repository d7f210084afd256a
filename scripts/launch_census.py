"""Kernel-launch census of a BASELINE workload sequence (GPU): launches and
device ms per kernel class for the first n_sw systems (rGCROT in the hybrid)
and for the whole sequence, next to the Krylov matvec counts.  Diagnostic
only (not part of the bench)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_03358_b200 as rk  # noqa: E402
from problems import get_workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = get_workload(name)
prob = w.problem()
prm = w.params
ctx = rk.Context(0)
dev = lambda a: torch.from_numpy(a).cuda()
rhs = lambda t: dev(prob.rhs(t).reshape(-1))
for n in (max(prm.n_sw, 1), w.n_systems):
    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets, dev(prob.bands(epoch=w.epoch(0))),
                         prob.periodic)
    s = rk.Solver(op, rk.config_from_params(prm, prm.method))
    xs = [torch.zeros(prob.N, dtype=torch.float64, device="cuda") for _ in range(n)]
    ctx.profile(True, None)
    ctx.profile_read(reset=True)
    reps = rk.solve_sequence(s, rhs, n, prm.method, n_sw=prm.n_sw, epoch_of=w.epoch,
                             bands_for_epoch=lambda e: dev(prob.bands(epoch=e)), x_out=xs)
    prof = ctx.profile_read()
    ctx.profile_read(reset=True)
    ctx.profile(False)
    print(f"== first {n} systems: tags {[r['tag'] for r in reps]}")
    print("   matvecs", [r["krylov_matvecs"] for r in reps], "total", sum(r["krylov_matvecs"] for r in reps))
    print("   operator_applications", [r.get("operator_applications") for r in reps])
    print("   cycles_or_iters", [r["cycles_or_iters"] for r in reps])
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"   {k:24s} {v['launches']:8d} {v['ms']:10.3f} ms")
    s.close()
    op.close()
