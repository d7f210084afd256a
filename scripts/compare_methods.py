"""Method comparison harness: GMRES(m), BiCGStab,
rGCROT(m,k) and the hybrid rGCROT -> rBiCGStab on one BASELINE workload,
all through librk on one GPU, reporting what the paper's tables report:
Krylov matvecs per system and solve time per system (`tab:turb1`,
`tab:porous1`, P:816-834 / P:1003-1019), plus the two central ratios
(recycling vs its base method).

    python scripts/compare_methods.py --workload c3 [--methods gmres,bicgstab,rgcrot,hybrid]

The paper's own numbers (CPU, GenIDLEST problems not available here) are
quoted as context only: porous medium, Jacobi, 10 steps -- BiCGStab 1480,
GMRES(30) 1800, rGCROT(10,40) 420, hybrid(5) 454 matvecs/step.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(workload, methods, out):
    import paper_1501_03358_b200 as rk
    from problems import get_workload
    w = get_workload(workload)
    prm = w.params
    prob = w.problem()
    ctx = rk.Context(0)
    stream = torch.cuda.current_stream()
    bands = torch.from_numpy(prob.bands(epoch=w.epoch(0))).cuda()
    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets, bands, prob.periodic)
    T = w.n_systems
    B = [torch.from_numpy(prob.rhs(t).reshape(-1)).cuda() for t in range(T)]
    X = [torch.zeros(prob.N, dtype=torch.float64, device="cuda") for _ in range(T)]
    epoch_bands = {}

    def bands_for(e):
        if e not in epoch_bands:
            epoch_bands[e] = torch.from_numpy(prob.bands(epoch=e)).cuda()
        return epoch_bands[e]

    res = {}
    for meth in methods:
        s = rk.Solver(op, rk.config_from_params(prm, meth))
        if w.epoch(0) != w.epoch(T - 1):
            op.update_bands(bands_for(w.epoch(0)))
        seq = lambda: rk.solve_sequence(s, lambda t: B[t], T, meth, n_sw=prm.n_sw, epoch_of=w.epoch,
                                        bands_for_epoch=bands_for, x_out=X)
        seq()                                   # warm-up (also fills the recycle space path)
        s.recycle_set(None)
        if w.epoch(0) != w.epoch(T - 1):
            op.update_bands(bands_for(w.epoch(0)))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        reps = seq()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        mv = [r["krylov_matvecs"] for r in reps]
        res[meth] = {"ms_per_system": ms / T, "krylov_matvecs_per_system": float(np.mean(mv)),
                     "matvecs": mv, "outcomes": sorted(set(r["outcome"] for r in reps)),
                     "ms_per_matvec": ms / max(1, sum(mv))}
        print(f"{meth:9s} {ms / T:9.2f} ms/system  {np.mean(mv):7.1f} matvecs/system  "
              f"{ms / max(1, sum(mv)):6.3f} ms/matvec  {res[meth]['outcomes']}", flush=True)
        s.close()
    ratios = {}
    if "rgcrot" in res and "gmres" in res:
        ratios["rgcrot_vs_gmres_matvecs"] = res["rgcrot"]["krylov_matvecs_per_system"] / res["gmres"]["krylov_matvecs_per_system"]
        ratios["rgcrot_vs_gmres_time"] = res["rgcrot"]["ms_per_system"] / res["gmres"]["ms_per_system"]
    if "hybrid" in res and "bicgstab" in res:
        ratios["hybrid_vs_bicgstab_matvecs"] = res["hybrid"]["krylov_matvecs_per_system"] / res["bicgstab"]["krylov_matvecs_per_system"]
        ratios["hybrid_vs_bicgstab_time"] = res["hybrid"]["ms_per_system"] / res["bicgstab"]["ms_per_system"]
    line = {"workload": workload, "description": w.description, "m": prm.m, "k": prm.k_max,
            "systems": T, "gpu": torch.cuda.get_device_name(0), "methods": res, "ratios": ratios,
            "paper_context": "porous (P:1011-1015, CPU x16 MPI, Jacobi): BiCGStab 1480, GMRES(30) 1800, "
                             "rGCROT(10,40) 420, hybrid(5) 454 matvecs/step"}
    print(json.dumps(ratios))
    if out:
        json.dump(line, open(out, "w"), indent=1)
    op.close()
    ctx.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--methods", default="gmres,bicgstab,rgcrot,hybrid")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    run(a.workload, a.methods.split(","), a.out)
