"""Per-rank kernel rate at z-slab sizes, on ONE GPU (no communication):
the compute side of strong scaling.  For a BASELINE workload and R ranks,
build the operator of one interior z-slab (planes [nz/2, nz/2 + nz/R) of
the global grid, z made non-periodic: cut faces contribute 0) as a
one-rank problem and run the workload's solver on it for a few systems;
report device ms per Krylov matvec next to the full grid's ms per matvec
/ R.  Convergence on the cut slab is not the point (a system may end
MAX_MATVECS): every Krylov matvec launches the same kernels, on the same
number of cells, as one rank of R does between its collectives.
usage: python scripts/slab_rate.py c4|c5 [R ...]  ->  one JSON line per R"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1501_03358_b200 as rk  # noqa: E402
from problems import get_workload  # noqa: E402

wname = sys.argv[1] if len(sys.argv) > 1 else "c4"
Rs = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
w = get_workload(wname)
prob, prm = w.problem(), w.params
ctx = rk.Context(0)
stream = torch.cuda.current_stream()
NSYS, WARM = (4, 2) if wname == "c4" else (6, 4)      # hybrid: the switch is after 3 systems
for R in Rs:
    nzl = prob.nz // R
    z0 = (prob.nz // 2) if R > 1 else 0
    z0 = min(z0, prob.nz - nzl)
    hb = prob.bands(z0, z0 + nzl)
    if R > 1:                      # cut faces: couplings out of the slab are dropped
        for d, (_, _, dz) in enumerate(np.asarray(prob.offsets)):
            if dz < 0:
                hb[d, 0] = 0.0
            elif dz > 0:
                hb[d, -1] = 0.0
    bands = torch.from_numpy(hb).cuda()
    periodic = prob.periodic if R == 1 else (prob.periodic & ~4)
    op = rk.GridOperator(ctx, prob.nx, prob.ny, nzl, prob.offsets, bands, periodic)
    cfg = rk.config_from_params(prm)
    s = rk.Solver(op, cfg)
    g = torch.Generator(device="cuda").manual_seed(7)
    B = [torch.rand(op.N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1 for _ in range(NSYS)]
    reps = rk.solve_sequence(s, lambda t: B[t], WARM, prm.method, n_sw=prm.n_sw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    reps = rk.solve_sequence(s, lambda t: B[t], NSYS - WARM, prm.method, n_sw=prm.n_sw, start=WARM)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    mv = sum(r["krylov_matvecs"] for r in reps)
    print(json.dumps({"workload": wname, "ranks": R, "slab": [prob.nx, prob.ny, nzl],
                      "tags": [r["tag"] for r in reps], "outcomes": [r["outcome"] for r in reps],
                      "krylov_matvecs": mv, "ms": round(ms, 2), "ms_per_matvec": round(ms / mv, 4)}), flush=True)
    s.close()
    op.close()
    del bands, B
    torch.cuda.empty_cache()
