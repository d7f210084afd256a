"""Oracle prefixes of the full-size configs (SURVEY §8(d) "c4: first 2 cycles
of system 0, plus 10 rBiCGStab iterations"; c5: the first cycle), stored for
the GPU parity test tests/gpu/test_gpu_prefix.py.  Only oracle/ and
problems/ are used (a stored value is written by a committed script that
calls only oracle/).  Writes tests/golden/oracle_prefix_<name>.json:

  rgcrot:     system 0 of the workload from an empty recycle space, x0 = 0,
              `cycles` rGCROT(m, k) cycles (tol = 1e-300): per cycle rho,
              H_ and B (the Arnoldi / projection coefficients), y; x after
              the last cycle as 4 seeded probe projections + 64 samples.
  rbicgstab:  system 1 with a k-column recycle space built by line 1b's
              refresh (C R = qr(A U0), reading D3) from U0[:, j] =
              problems.rng.uniform(5000 + j, n); `iters` iterations: per
              iteration rho, sigma, ||s||^2, t^T s, t^T t, ||r||^2, ||v||^2;
              x after line 17a as above.

    python scripts/oracle_prefix.py c4      # ~30 min on 8 cores, ~15 GB
    python scripts/oracle_prefix.py c5      # ~10 min, ~30 GB
"""
import json
import os
import sys
import time
from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.krylov import rbicgstab, refresh_space, rgcrot  # noqa: E402
from oracle.stencil import Jacobi, Operator  # noqa: E402
from problems import get_workload  # noqa: E402
from problems.rng import uniform  # noqa: E402

PLAN = {"c4": {"cycles": 2, "iters": 10}, "c5": {"cycles": 1, "iters": 0}}
NPROBE, NSAMPLE = 4, 64


def xsummary(x):
    N = x.size
    idx = np.arange(N, dtype=np.uint64)
    sidx = [int(i) for i in np.linspace(0, N - 1, NSAMPLE).round()]
    return {"xnorm": float(np.linalg.norm(x)), "xmax": float(np.abs(x).max()),
            "xproj": [float(uniform(7000 + q, idx) @ x) for q in range(NPROBE)],
            "sample_idx": sidx, "xsample": [float(x[i]) for i in sidx]}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    plan = PLAN[name]
    w = get_workload(name)
    prm = w.params
    prob = w.problem()
    t0 = time.time()
    op = Operator.from_problem(prob)
    pc = Jacobi(op, prm.sweeps, prm.omega_l, prm.omega_g)
    out = {"workload": name, "description": w.description, "m": prm.m, "k_max": prm.k_max,
           "generated_by": "python scripts/oracle_prefix.py " + name}
    # rGCROT prefix of system 0
    cyc = []
    b0 = prob.rhs(0).reshape(-1)
    e = np.zeros((op.N, 0))
    p = replace(prm, method="rgcrot", max_mv=plan["cycles"] * prm.m, tol=1e-300)
    x, U, C, rep = rgcrot(op, pc, b0, e, e, p, hook=lambda d: cyc.append(
        {"k": int(d["B"].shape[0]), "m_eff": int(d["m_eff"]), "rho": float(d["rho"]),
         "H": d["H"].T.tolist(), "B": d["B"].T.tolist(), "y": d["y"].tolist()}))
    print("rgcrot", rep.krylov_mv, "matvecs", round(time.time() - t0, 1), "s", flush=True)
    out["rgcrot"] = {"system": 0, "krylov_matvecs": int(rep.krylov_mv), "cycles": cyc,
                     **xsummary(x), "note": "H and B stored row = column j (transposed)"}
    del U, C, x
    if plan["iters"]:
        k = prm.k_max
        n = np.arange(op.N, dtype=np.uint64)
        U0 = np.column_stack([uniform(5000 + j, n) for j in range(k)])
        Ur, Cr, _ = refresh_space(op.apply, U0)
        del U0
        b1 = prob.rhs(1).reshape(-1)
        its = []
        p = replace(prm, method="rbicgstab", max_mv=2 * plan["iters"], tol=1e-300, k_max=k + 2)
        x, _, _, rep = rbicgstab(op, pc, b1, Ur, Cr, p, hook=lambda d: its.append(
            {q: float(d[q]) for q in ("rho", "sigma", "ss", "ts", "tt", "rr", "vv")}))
        r0 = b1 - Cr @ (Cr.T @ b1)
        print("rbicgstab", rep.krylov_mv, "matvecs", round(time.time() - t0, 1), "s", flush=True)
        out["rbicgstab"] = {"system": 1, "k": k, "u0_seeds": [5000, 5000 + k - 1],
                            "krylov_matvecs": int(rep.krylov_mv), "r0norm": float(np.linalg.norm(r0)),
                            "iterations": its, **xsummary(x)}
    out["cpu_seconds"] = round(time.time() - t0, 1)
    path = os.path.join(ROOT, "tests", "golden", f"oracle_prefix_{name}.json")
    json.dump(out, open(path, "w"))
    print("wrote", path, out["cpu_seconds"], "s")


if __name__ == "__main__":
    main()
