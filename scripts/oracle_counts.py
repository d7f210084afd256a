"""Run the CPU oracle over a whole BASELINE workload sequence and store what
the GPU parity tests and bench.py's reference arm compare against.

Writes tests/golden/oracle_seq_<name>.json: per system the method tag, the
Krylov matvec count, operator applications, cycles/iterations, outcome, the
true relative residual, ||x_t|| and x_t's projections on 4 seeded probe
vectors (problems.rng, seeds 7000+q) plus 64 sampled entries -- enough for
solution parity at full size without storing x.  Only oracle/ and problems/
are used (a stored value is written by a committed script that
calls only oracle/).

    python scripts/oracle_counts.py c3        # ~25 min on 8 cores
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import run_sequence  # noqa: E402
from problems import get_workload  # noqa: E402
from problems.rng import uniform  # noqa: E402

NPROBE = 4
NSAMPLE = 64


def probes(N):
    idx = np.arange(N, dtype=np.uint64)
    return [uniform(7000 + q, idx) for q in range(NPROBE)]


def sample_idx(N):
    return [int(i) for i in np.linspace(0, N - 1, NSAMPLE).round()]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    solver = sys.argv[2] if len(sys.argv) > 2 else None
    w = get_workload(name)
    prob = w.problem()
    g = probes(prob.N)
    sidx = sample_idx(prob.N)
    rows = []
    t0 = time.time()

    def cb(t, tag, x, U, C, rep):
        b = prob.rhs(t).reshape(-1)
        rows.append({
            "t": t, "tag": tag, "krylov_matvecs": int(rep.krylov_mv),
            "operator_applications": int(rep.op_apps), "cycles_or_iters": int(rep.cycles),
            "bnorm": float(rep.bnorm),
            "outcome": int(rep.outcome), "true_rel_res": float(rep.final_true_res / np.linalg.norm(b)),
            "xnorm": float(np.linalg.norm(x)), "xproj": [float(gq @ x) for gq in g],
            "xsample": [float(x[i]) for i in sidx], "k_after": int(U.shape[1]),
            "elapsed_s": round(time.time() - t0, 1)})
        print(json.dumps({k: rows[-1][k] for k in ("t", "tag", "krylov_matvecs", "outcome",
                                                   "true_rel_res", "elapsed_s")}), flush=True)

    run_sequence(w, solver=solver, callback=cb)
    out = {"workload": name, "solver": solver or w.params.method, "description": w.description,
           "generated_by": "python scripts/oracle_counts.py " + " ".join(sys.argv[1:]),
           "probe_seeds": [7000 + q for q in range(NPROBE)], "sample_idx": sidx,
           "cpu_seconds": round(time.time() - t0, 1), "systems": rows}
    suffix = "" if solver is None else "_" + solver
    path = os.path.join(ROOT, "tests", "golden", f"oracle_seq_{name}{suffix}.json")
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
