"""Collective launches per Krylov step of librk's multi-rank schedule
(rk_comm_count), measured on one GPU through the in-process rank group:
prints, per system of a workload on R z-slabs, the all-reduce and halo
launches next to the Krylov matvecs and cycles / iterations.
usage: python scripts/count_collectives.py [workload] [R] [force_chain]"""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
wname = sys.argv[1] if len(sys.argv) > 1 else "c2m"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if len(sys.argv) > 3 and sys.argv[3] == "1":
    os.environ["RK_FORCE_CHAIN"] = "1"
import paper_1501_03358_b200 as rk  # noqa: E402
from problems import get_workload, slab_range  # noqa: E402

w = get_workload(wname)
prob, prm, T = w.problem(), w.params, w.n_systems
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
uid = ("RKLOCAL:count_" + wname).encode().ljust(128, b"\0")
out = [None] * R


def rank(r):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        z0, z1 = slab_range(prob.nz, r, R)
        ctx = rk.Context(0, r, R, uid=uid, stream=st.cuda_stream)
        op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets,
                             dev(prob.bands(z0, z1, epoch=w.epoch(0))), prob.periodic, z0=z0, nz_local=z1 - z0)
        s = rk.Solver(op, rk.config_from_params(prm))
        rows = []
        for t in range(T):
            a0, h0 = ctx.comm_count()
            rep = rk.solve_sequence(s, lambda q: dev(prob.rhs(q, z0, z1).reshape(-1)), 1, prm.method,
                                    n_sw=prm.n_sw, epoch_of=w.epoch,
                                    bands_for_epoch=lambda e: dev(prob.bands(z0, z1, epoch=e)), start=t)[0]
            a1, h1 = ctx.comm_count()
            rows.append((rep["tag"], rep["krylov_matvecs"], rep["operator_applications"],
                         rep["cycles_or_iters"], a1 - a0, h1 - h0))
        st.synchronize()
        out[r] = rows
        s.close(); op.close(); ctx.close()


th = [threading.Thread(target=rank, args=(r,)) for r in range(R)]
[t.start() for t in th]
[t.join() for t in th]
assert all(o == out[0] for o in out)
print(wname, "R =", R, "m =", prm.m, "k =", prm.k_max)
print("tag matvecs op_apps cycles/iters allreduces halos | allreduces/matvec halos/op_app")
for tag, mv, oa, cy, a, h in out[0]:
    print(tag, mv, oa, cy, a, h, "|", round(a / max(mv, 1), 3), round(h / max(oa, 1), 3))
