"""Diagnose the c4 hybrid's MAX_MATVECS systems with
the ORACLE alone: run a c4-shaped sequence (19-point channel, A perturbed
every 10 systems, rGCROT(40,30) then rBiCGStab with the frozen space) at
64^3 and record per-system outcome, Krylov matvecs and tags.  If the oracle
also fails to converge on post-epoch rBiCGStab systems the failure is the
method's behaviour on this synthetic sequence, not a librk bug.

    python scripts/diag_c4h.py c4hm [policy]      # policy: refresh_on_epoch | switchback
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import run_sequence  # noqa: E402
from oracle.krylov import OUTCOME_NAMES  # noqa: E402
from problems import get_workload  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4hm"
    policy = sys.argv[2] if len(sys.argv) > 2 else ""
    w = get_workload(name)
    kw = {policy: True} if policy else {}
    rows = []
    t0 = time.time()

    def cb(t, tag, x, U, C, rep):
        rows.append({"t": t, "epoch": w.epoch(t), "tag": tag, "outcome": OUTCOME_NAMES[rep.outcome],
                     "krylov_matvecs": int(rep.krylov_mv), "k_after": int(U.shape[1]),
                     "true_rel_res": float(rep.final_true_res / rep.bnorm),
                     "elapsed_s": round(time.time() - t0, 1)})
        print(json.dumps(rows[-1]), flush=True)

    run_sequence(w, callback=cb, **kw)
    out = {"workload": name, "policy": policy or "none", "description": w.description,
           "generated_by": "python scripts/diag_c4h.py " + " ".join(sys.argv[1:]), "systems": rows}
    path = os.path.join(ROOT, "profiles", "r02_c4h_diag", f"oracle_{name}{'_' + policy if policy else ''}.json")
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
