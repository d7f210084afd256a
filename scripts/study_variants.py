"""Variant study on one
BASELINE workload, through librk on one GPU: truncation T1 (drop the oldest,
SPEC S:285) vs T2 (principal angles, the GCROT criterion P:460-465,
DESIGN.md R13), and the hybrid rGCROT -> rBiCGStab plain, with the
intermittent rGCROT solve at every A epoch ("when the system matrix
changes", refresh_on_epoch) and with switch-back on poor
convergence, next to plain BiCGStab / GMRES.  One timed pass
over the whole sequence per variant (device time), per-system Krylov
matvecs, outcomes and method tags.

    python scripts/study_variants.py --workload c4 \
        --variants rgcrot:T1,rgcrot:T2,hybrid,hybrid+refresh_on_epoch,hybrid+switchback,bicgstab
"""
import argparse
import json
import os
import sys
from dataclasses import replace

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse_variant(v):
    meth, _, rest = v.partition(":")
    meth, _, policy = meth.partition("+")
    return meth, (rest or "T1"), policy


def main():
    import paper_1501_03358_b200 as rk
    from problems import get_workload
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--variants", default="rgcrot:T1,rgcrot:T2,hybrid,hybrid+refresh_on_epoch,"
                                          "hybrid+switchback,bicgstab")
    ap.add_argument("--systems", type=int, default=0)
    ap.add_argument("--outdir", default=os.path.join(ROOT, "profiles", "r02_compare"))
    a = ap.parse_args()
    os.makedirs(a.outdir, exist_ok=True)
    w = get_workload(a.workload)
    prob = w.problem()
    T = a.systems or w.n_systems
    ctx = rk.Context(0)
    stream = torch.cuda.current_stream()
    epoch_bands = {}

    def bands_for(e):
        if e not in epoch_bands:
            epoch_bands[e] = torch.from_numpy(prob.bands(epoch=e)).cuda()
        return epoch_bands[e]

    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets, bands_for(w.epoch(0)),
                         prob.periodic)
    B = [torch.from_numpy(prob.rhs(t).reshape(-1)).cuda() for t in range(T)]
    X = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
    if prob.N <= (1 << 21):   # small grids: one untimed pass first (launch set-up, occupancy queries)
        s = rk.Solver(op, rk.config_from_params(w.params))
        rk.solve_sequence(s, lambda t: B[t], min(T, 2), w.params.method, n_sw=w.params.n_sw,
                          epoch_of=w.epoch, bands_for_epoch=bands_for, x_out=[X] * T)
        s.close()
    for v in a.variants.split(","):
        meth, trunc, policy = parse_variant(v)
        prm = replace(w.params, trunc=trunc)
        s = rk.Solver(op, rk.config_from_params(prm, meth))
        op.update_bands(bands_for(w.epoch(0)))
        kw = {policy: True} if policy else {}
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        reps = rk.solve_sequence(s, lambda t: B[t], T, meth, n_sw=prm.n_sw, epoch_of=w.epoch,
                                 bands_for_epoch=bands_for, x_out=[X] * T, **kw)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        mv = [r["krylov_matvecs"] for r in reps]
        bad = [t for t, r in enumerate(reps) if r["outcome"] != "CONVERGED"]
        res = {"workload": a.workload, "description": w.description, "variant": v, "method": meth,
               "trunc": trunc, "policy": policy or "none", "m": prm.m, "k": prm.k_max, "k_t": prm.k_t,
               "p1": prm.p1, "n_sw": prm.n_sw, "systems": T, "ms_per_system": ms / T,
               "krylov_matvecs_per_system": float(np.mean(mv)), "ms_per_matvec": ms / max(1, sum(mv)),
               "matvecs": mv, "outcomes": [r["outcome"] for r in reps], "tags": [r["tag"] for r in reps],
               "not_converged": bad, "k_after": [r["k_after"] for r in reps],
               "gpu": torch.cuda.get_device_name(0)}
        print(f"{a.workload} {v:28s} {ms / T:9.1f} ms/system {np.mean(mv):7.1f} mv/system "
              f"not converged: {bad}", flush=True)
        name = v.replace(":", "_").replace("+", "_")
        json.dump(res, open(os.path.join(a.outdir, f"{a.workload}_{name}.json"), "w"), indent=1)
        s.close()
    op.close()
    ctx.close()


if __name__ == "__main__":
    main()
