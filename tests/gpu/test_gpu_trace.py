"""Per-step parity at the north star's 1e-12 (reading D25: componentwise,
scaled by the magnitudes the quantity is formed from).  librk's rk_trace
returns the values its kernels produced at every rGCROT cycle (rho, the
Hessenberg H_ from the Arnoldi block dots and updates, the recycle
projections B = C^T w, the least-squares y; PAPER Alg. 3 lines 4-12,
P:313-323) and every rBiCGStab iteration (rho, sigma, ||s||^2, t^T s,
t^T t, ||r||^2; Alg. 4 lines 4-15), so the block-dot, block-
update, Gram-corrected CGS2, projection, bicg_* and chain kernels are
compared one step at a time with the oracle run from the same start (a
recycle space the ORACLE built: random U, line-1a refresh).

GPU orthogonalisation: its default Gram-corrected CGS2 (R19) and plain
CGS2; oracle: textbook CGS2 (the coefficients agree to rounding, R19)."""
from dataclasses import replace

import numpy as np
import pytest
import torch

from oracle.krylov import rbicgstab, refresh_space, rgcrot
from oracle.stencil import Jacobi, Operator
from problems import get_workload
from problems.stencils import channel19, porous7

from bicg_check import TOL, check_bicg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1501_03358_b200 as rk
    rk.lib()
    return rk


@pytest.fixture(scope="module")
def ctx(rk):
    c = rk.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def oracle_space(op, apply, k, seed):
    U0 = np.random.default_rng(seed).uniform(-1, 1, (op.N, k))
    U, C, _ = refresh_space(apply, U0)
    assert U.shape[1] == k
    return U, C


def gpu_run(rk, ctx, prob, prm, method, U, C, b, gpu_ortho=None):
    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets, dev(prob.bands()),
                         prob.periodic)
    cfg = rk.config_from_params(prm, method) if gpu_ortho is None else \
        rk.config_from_params(prm, method, ortho=gpu_ortho)
    s = rk.Solver(op, cfg)
    s.recycle_set(dev(U.T), dev(C.T))
    x, rep = s.solve(dev(b), tol=1e-300)
    cyc, bi = s.trace()
    s.close()
    op.close()
    return x.cpu().numpy(), rep, cyc, bi


CYCLE_CASES = [
    ("channel16", lambda: channel19(16), 12, 6),
    ("porous24", lambda: porous7(24, 3), 8, 8),
    ("channel32", lambda: channel19(32), 20, 10),
    ("c3_full", lambda: porous7(128, 6), 10, 20),
]


@pytest.mark.parametrize("gpu_ortho", [None, "cgs2"], ids=["gram_cgs2", "cgs2"])
@pytest.mark.parametrize("name,mk,m,k", CYCLE_CASES, ids=[c[0] for c in CYCLE_CASES])
def test_rgcrot_cycle_trace(rk, ctx, name, mk, m, k, gpu_ortho):
    """Two rGCROT(m, k) cycles from the same recycle space: rho, every
    column of H_ and B to 1e-12 of that column's norm (|[B; H_](:, j)| is
    the norm of the vector the block dot / update / normalisation kernels
    orthogonalised), the least-squares y to 1e-12 cond(H_), and x."""
    prob = mk()
    op = Operator.from_problem(prob)
    pc = Jacobi(op)
    U, C = oracle_space(op, lambda v: pc(op.apply(v)), k, 41)
    b = prob.rhs(1).reshape(-1)
    prm = replace(get_workload("c2s").params, m=m, k_max=k + 2, k_t=k, p1=1, max_mv=2 * m,
                  tol=1e-300)
    ocyc = []
    xo, _, _, ro = rgcrot(op, pc, b, U.copy(), C.copy(), prm, hook=lambda d: ocyc.append(d))
    xg, rg, gcyc, _ = gpu_run(rk, ctx, prob, prm, "rgcrot", U, C, b, gpu_ortho)
    assert len(ocyc) == len(gcyc) == 2 and rg["krylov_matvecs"] == ro.krylov_mv
    for co, cg in zip(ocyc, gcyc):
        mo = co["m_eff"]
        assert cg["m_eff"] == mo and cg["k"] == co["B"].shape[0]
        assert abs(cg["rho"] - co["rho"]) <= TOL * co["rho"]
        HB_o = np.vstack([co["B"], co["H"]])
        HB_g = np.vstack([cg["B"], cg["H"]])
        scale = np.linalg.norm(HB_o, axis=0)
        err = np.abs(HB_g - HB_o).max(axis=0)
        assert np.all(err <= TOL * scale), (name, float((err / scale).max()))
        kap = np.linalg.cond(co["H"])
        dy = np.linalg.norm(cg["y"] - co["y"]) / np.linalg.norm(co["y"])
        assert dy <= TOL * max(1.0, kap), (name, dy, kap)
    kap = max(np.linalg.cond(c["H"]) for c in ocyc)
    assert np.linalg.norm(xg - xo) <= TOL * max(1.0, kap) * np.linalg.norm(xo)


BICG_CASES = [
    ("porous24", lambda: porous7(24, 3), 8),
    ("channel32", lambda: channel19(32), 10),
    ("c3_full", lambda: porous7(128, 6), 20),
]


@pytest.mark.parametrize("name,mk,k", BICG_CASES, ids=[c[0] for c in BICG_CASES])
def test_rbicgstab_iteration_trace(rk, ctx, name, mk, k):
    """Four rBiCGStab iterations with a k-dimensional space (C R = qr(A U),
    reading D3): rho = r~^T r to 1e-12 |r~||r|, sigma = r~^T v to
    1e-12 |r~||v|, t^T s to 1e-12 |t||s|, ||s||^2, t^T t, ||r||^2 to 1e-12
    relative, and x after line 17a."""
    prob = mk()
    op = Operator.from_problem(prob)
    pc = Jacobi(op)
    U, C = oracle_space(op, op.apply, k, 43)
    b = prob.rhs(2).reshape(-1)
    prm = replace(get_workload("c3s").params, k_max=k + 2, k_t=k, max_mv=8, tol=1e-300)
    oit = []
    xo, _, _, ro = rbicgstab(op, pc, b, U.copy(), C.copy(), prm, hook=lambda d: oit.append(d))
    xg, rg, _, bi = gpu_run(rk, ctx, prob, prm, "rbicgstab", U, C, b)
    assert rg["krylov_matvecs"] == ro.krylov_mv == 8 and len(oit) == len(bi) == 4
    r0 = np.linalg.norm(b - C @ (C.T @ b))
    check_bicg(bi, oit, r0)
    assert np.linalg.norm(xg - xo) <= TOL * 10 * np.linalg.norm(xo)
