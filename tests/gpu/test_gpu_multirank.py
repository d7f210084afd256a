"""librk's own multi-rank schedule on one GPU (VERDICT r01 next-round item 6:
"a CPU test that drives librk's own halo/allreduce schedule").  R ranks are
R contexts of this process, each driven by its own host thread and CUDA
stream, joined into an in-process rank group ("RKLOCAL:<name>" uid,
comm.cpp): every halo() and allreduce() that the solvers issue -- in the
order they issue them -- runs, with the halo as a device copy of the
neighbour's boundary plane after the neighbour's producer event and the
all-reduce summed on the host in rank order.  No rank's kernel ever waits
on another rank's kernel.  The slab data paths (z-slab ghost planes,
periodic-z rings, block-Jacobi blocks without halo, multi-rank reduction
finalisation without the one-rank fusions) are the product code.

With RK_FORCE_CHAIN the fused TMA chains run on the slabs too: one
NST-deep halo exchange of the chain input (and of the sweeps' right-hand
side) per launch, the neighbours' band planes from the ghost-band copy made
at rk_op_create.

Checks, at world 2 and 3:
  * SpMV and M^-1 on slabs == the one-rank result bit for bit (no
    reductions involved; reading R17 block Jacobi with one block per rank),
    unfused and through the fused 7- and 19-point chains;
  * whole solve sequences: every rank reports the same outcomes, counts
    and residuals, and returns the same per-cycle Krylov state (rk_trace,
    bit for bit: the replicated H, B, y of SURVEY §8(e)); the stitched
    solution matches the oracle under the usual parity tolerances."""
import threading

import numpy as np
import pytest
import torch

from oracle import run_sequence
from problems import OFFSETS7, OFFSETS19, get_workload, slab_range
from problems.stencils import StencilProblem

from test_gpu_parity import compare_sequences, random_op_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1501_03358_b200 as rk
    rk.lib()
    return rk


def uid(name):
    b = ("RKLOCAL:" + name).encode()
    return b + b"\0" * (128 - len(b))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def run_ranks(R, fn, timeout=600):
    out = [None] * R
    errs = []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:   # noqa: BLE001 -- reported below
            errs.append((r, e))

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "a rank did not finish (deadlocked schedule?)"
    assert not errs, errs
    return out


def slab_op(rk, prob, r, R, name, st, epoch=0):
    z0, z1 = slab_range(prob.nz, r, R)
    ctx = rk.Context(0, r, R, uid=uid(name), stream=st.cuda_stream)
    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets,
                         dev(prob.bands(z0, z1, epoch=epoch)), prob.periodic, z0=z0, nz_local=z1 - z0)
    return ctx, op, z0, z1


def _random_problem(nx, ny, nz, periodic, offsets, seed):
    bands = random_op_problem(nx, ny, nz, periodic, offsets, seed)
    return StencilProblem(name="random", nx=nx, ny=ny, nz=nz, periodic=periodic,
                          offsets=np.asarray(offsets), _band_fn=lambda z0, z1: bands[:, z0:z1].copy())


PROBLEMS = {
    "c4_full": lambda: get_workload("c4").problem(),
    "c3_full": lambda: get_workload("c3").problem(),
    "c3s": lambda: get_workload("c3s").problem(),
    "c2s": lambda: get_workload("c2s").problem(),
    "rand7_64x32x48": lambda: _random_problem(64, 32, 48, 0, OFFSETS7, 31),
    "rand7_64x32x48_pz": lambda: _random_problem(64, 32, 48, 4, OFFSETS7, 32),
    "rand19_64x16x40_pxz": lambda: _random_problem(64, 16, 40, 5, OFFSETS19, 33),
    "rand19_32x24x48": lambda: _random_problem(32, 24, 48, 0, OFFSETS19, 34),
}


@pytest.mark.parametrize("wname,R,force", [
    ("c4_full", 2, False), ("c3_full", 4, False),      # full size: the chains by the L2 rule
    ("c3s", 2, False), ("c3s", 3, False), ("c2s", 2, False), ("c2s", 3, False),
    ("rand7_64x32x48", 2, True), ("rand7_64x32x48", 3, True), ("rand7_64x32x48_pz", 2, True),
    ("rand19_64x16x40_pxz", 2, True), ("rand19_32x24x48", 3, True)])
def test_slab_operator_and_preconditioner_bitwise(rk, wname, R, force, monkeypatch):
    prob = PROBLEMS[wname]()
    if force:
        monkeypatch.setenv("RK_FORCE_CHAIN", "1")     # read at rk_op_create
    x = np.random.default_rng(5).uniform(-1, 1, prob.N)
    ctx1 = rk.Context(0)
    op1 = rk.GridOperator(ctx1, prob.nx, prob.ny, prob.nz, prob.offsets, dev(prob.bands()), prob.periodic)
    y1 = op1.apply(dev(x)).cpu().numpy()
    z1 = op1.precond(dev(x)).cpu().numpy()
    zb1 = op1.precond(dev(x), zblocks=R).cpu().numpy() if prob.nz % R == 0 else None
    op1.close()
    ctx1.close()
    P = prob.nx * prob.ny

    def rank(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx, op, za, zb = slab_op(rk, prob, r, R, f"op_{wname}_{R}", st)
            xs = dev(x[za * P:zb * P])
            y = op.apply(xs).cpu().numpy()
            z = op.precond(xs).cpu().numpy()
            zbl = op.precond(xs, zblocks=R).cpu().numpy() if prob.nz % R == 0 else None
            st.synchronize()
            op.close()
            ctx.close()
            return y, z, zbl

    res = run_ranks(R, rank)
    monkeypatch.delenv("RK_FORCE_CHAIN", raising=False)
    assert np.array_equal(np.concatenate([r[0] for r in res]), y1)
    assert np.array_equal(np.concatenate([r[1] for r in res]), z1)
    if zb1 is not None:
        assert np.array_equal(np.concatenate([r[2] for r in res]), zb1)


@pytest.mark.parametrize("wname,R,force", [("c3s", 2, False), ("c3s", 3, False), ("c2s", 2, False),
                                           ("c2s", 3, False), ("c4hs", 2, False), ("c2m", 2, True)])
def test_slab_sequence_replicated_state(rk, wname, R, force, monkeypatch):
    w = get_workload(wname)
    if force:
        monkeypatch.setenv("RK_FORCE_CHAIN", "1")
    prob = w.problem()
    prm = w.params
    T = w.n_systems

    def rank(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx, op, z0, z1 = slab_op(rk, prob, r, R, f"seq_{wname}_{R}", st, epoch=w.epoch(0))
            s = rk.Solver(op, rk.config_from_params(prm))
            xs = [torch.zeros(op.N, dtype=torch.float64, device="cuda") for _ in range(T)]
            traces = []
            reps = []
            for t in range(T):   # one call per system to collect each system's trace
                reps += rk.solve_sequence(s, lambda q: dev(prob.rhs(q, z0, z1).reshape(-1)), 1,
                                          prm.method, n_sw=prm.n_sw, epoch_of=w.epoch,
                                          bands_for_epoch=lambda e: dev(prob.bands(z0, z1, epoch=e)),
                                          x_out=[xs[t]], start=t)
                traces.append(s.trace())
            st.synchronize()
            out = (reps, [x.cpu().numpy() for x in xs], traces)
            s.close()
            op.close()
            ctx.close()
            return out

    res = run_ranks(R, rank)
    monkeypatch.delenv("RK_FORCE_CHAIN", raising=False)
    keys = ("outcome", "krylov_matvecs", "operator_applications", "cycles_or_iters", "k_after",
            "bnorm", "final_true_res", "final_updated_res", "tag")
    for r in range(1, R):
        for a, b in zip(res[0][0], res[r][0]):
            assert all(a[k] == b[k] for k in keys), (r, a, b)
        for (ca, ba), (cb, bb) in zip(res[0][2], res[r][2]):
            assert np.array_equal(ba, bb)
            assert len(ca) == len(cb)
            for u, v in zip(ca, cb):
                assert all(np.array_equal(u[q], v[q]) for q in ("H", "B", "y")) and u["rho"] == v["rho"]
    gpu = [(res[0][0][t], np.concatenate([res[r][1][t] for r in range(R)])) for t in range(T)]
    ora = run_sequence(w)
    compare_sequences(w, gpu, ora, prm.method)


def test_full_size_c4_solve_two_slabs_vs_one_rank(rk):
    """SURVEY §8(d) "GPU-vs-GPU parity: c4/c5 at P > 1 vs P = 1" at full size,
    on one GPU through the in-process rank group: system 0 of c4 (256^3
    19-point channel, rGCROT(40,30) T2 from an empty space) on 2 z-slabs of
    128 planes -- fused 19-point chains with deep halos and ghost bands,
    all-reduced reductions -- against the one-rank solve: both converge, the
    Krylov matvec counts agree within one cycle, and both solutions are
    certified solutions (true residual <= tol ||b||, recomputed here by the
    oracle's operator); they agree to 1e-4 relative -- the channel operator is
    ill-conditioned, so two tol-converged solutions may differ by more than the
    north star's 1e-6 (reading R12), and the reductions differ in order."""
    w = get_workload("c4")
    prob = w.problem()
    prm = w.params
    b = prob.rhs(0).reshape(-1)
    ctx1 = rk.Context(0)
    op1 = rk.GridOperator(ctx1, prob.nx, prob.ny, prob.nz, prob.offsets, dev(prob.bands()), prob.periodic)
    s1 = rk.Solver(op1, rk.config_from_params(prm))
    x1, r1 = s1.solve(dev(b))
    x1 = x1.cpu().numpy()
    s1.close()
    op1.close()
    ctx1.close()
    P = prob.nx * prob.ny

    def rank(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx, op, z0, z1 = slab_op(rk, prob, r, 2, "c4_full_solve", st)
            s = rk.Solver(op, rk.config_from_params(prm))
            x, rep = s.solve(dev(b[z0 * P:z1 * P]))
            st.synchronize()
            out = (rep, x.cpu().numpy())
            s.close()
            op.close()
            ctx.close()
            return out

    res = run_ranks(2, rank, timeout=1200)
    assert r1["outcome"] == "CONVERGED" and all(rep["outcome"] == "CONVERGED" for rep, _ in res)
    assert res[0][0]["krylov_matvecs"] == res[1][0]["krylov_matvecs"]
    assert abs(res[0][0]["krylov_matvecs"] - r1["krylov_matvecs"]) <= prm.m
    x2 = np.concatenate([x for _, x in res])
    from oracle.stencil import Operator
    A = Operator.from_problem(prob)
    bn = np.linalg.norm(b)
    for x in (x1, x2):
        assert np.linalg.norm(b - A.apply(x)) <= prm.tol * bn * (1 + 1e-6)
    assert np.linalg.norm(x2 - x1) <= 1e-4 * np.linalg.norm(x1)


@pytest.mark.parametrize("wname,force,halos_per_op", [("c2m", True, 3), ("c4hs", False, 6)])
def test_collectives_per_krylov_step(rk, wname, force, halos_per_op, monkeypatch):
    """SURVEY §8(e) / north_star: "allreduce for every dot product, batched so
    each iteration issues as few collectives as the algorithm allows".
    rk_comm_count counts collective launches the way NCCL issues them (a group
    counts once); on two z-slabs, per system:
      * rGCROT: 2 all-reduces per Arnoldi step ([C V_j]^T [w v_j] in one
        collective whatever the column count; ||w||^2) + 3 per cycle
        (line 1b / true residual / cycle-start norms) + <= 3 per solve;
      * rBiCGStab: exactly 4 per iteration + 10 per solve, + 6
        when the space is refreshed first;
      * halos: one launch per fused 19-point chain launch (3 per
        preconditioned operator: input and rhs halos grouped), 6 per
        operator on the unfused path (one plane per stencil application),
        plus a few per cycle / solve (true residual, M^-1 r, refresh)."""
    w = get_workload(wname)
    if force:
        monkeypatch.setenv("RK_FORCE_CHAIN", "1")
    prob, prm, T, R = w.problem(), w.params, w.n_systems, 2

    def rank(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx, op, z0, z1 = slab_op(rk, prob, r, R, f"coll_{wname}", st, epoch=w.epoch(0))
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
            s.close()
            op.close()
            ctx.close()
            return rows

    res = run_ranks(R, rank)
    monkeypatch.delenv("RK_FORCE_CHAIN", raising=False)
    assert res[0] == res[1]
    tags = set()
    for tag, mv, oa, cy, a, h in res[0]:
        tags.add(tag)
        if tag == "rgcrot":
            assert mv == prm.m * cy
            assert 2 * mv + 3 * cy <= a <= 2 * mv + 3 * cy + 3, (tag, mv, cy, a)
            assert halos_per_op * mv <= h <= halos_per_op * mv + (halos_per_op + 2) * cy + 8, (tag, mv, cy, h)
        else:
            assert mv == 2 * cy
            refreshed = oa > 1
            assert a == 4 * cy + 10 + (6 if refreshed else 0), (tag, cy, oa, a)
            assert halos_per_op * mv <= h <= halos_per_op * (mv + oa) + 16, (tag, mv, oa, h)
    assert tags == {"rgcrot", "rbicgstab"}
    # one rank: no collectives at all
    ctx1 = rk.Context(0)
    assert ctx1.comm_count() == (0, 0)
    ctx1.close()
