"""Pins for oracle O3-O7 against mathematics and library routines:
brute-force least squares over explicit spaces (eqs. (6)-(7), Alg. 1
line 12), scipy.sparse.linalg.bicgstab, dense direct solves, and the
algebraic invariants of eqs. (4), (5), (8)."""
from dataclasses import replace

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle.krylov import (
    BREAKDOWN, CONVERGED, gcrot_update, bicgstab, gmres, rbicgstab,
    refresh_space, rgcrot, run_sequence,
)
from oracle.stencil import Jacobi, Operator, to_dense
from problems import OFFSETS7, SolverParams, get_workload
from problems.stencils import channel19, convection_diffusion_c1, porous7


def _setup(prob, seed=0):
    op = Operator.from_problem(prob)
    pc = Jacobi(op)
    b = prob.rhs(1).reshape(-1)
    return op, pc, b


def _Ahat_dense(op, pc):
    D = to_dense(op)
    return np.column_stack([pc(D[:, i]) for i in range(op.N)]), D


def _orth(M):
    q, _ = np.linalg.qr(M)
    return q


def test_gmres_one_cycle_is_minimal_residual():
    """Alg. 1 line 12: after one cycle from x0 = 0, x minimises
    ||M^-1 b - A_hat x|| over K_m(A_hat, M^-1 b).  Brute force: explicit
    (QR-orthonormalised) power basis + numpy lstsq."""
    prob = convection_diffusion_c1(5)
    op, pc, b = _setup(prob)
    m = 6
    prm = SolverParams(m=m, k_max=0, p1=0, tol=1e-30, max_mv=m)
    x, rep = gmres(op, pc, b, prm)
    assert rep.cycles == 1 and rep.krylov_mv == m
    Ah, _ = _Ahat_dense(op, pc)
    rh = pc(b)
    K = [rh]
    for _ in range(m - 1):
        K.append(Ah @ K[-1])
    Q = _orth(np.column_stack(K))
    c = np.linalg.lstsq(Ah @ Q, rh, rcond=None)[0]
    xb = Q @ c
    assert np.linalg.norm(x - xb) <= 1e-9 * np.linalg.norm(xb)


def test_gmres_finite_termination_and_identity():
    prob = convection_diffusion_c1(3)                     # N = 27
    op, pc, b = _setup(prob)
    prm = SolverParams(m=27, k_max=0, p1=0, tol=1e-10)
    x, rep = gmres(op, pc, b, prm)
    assert rep.outcome == CONVERGED and rep.cycles == 1
    xs = np.linalg.solve(to_dense(op), b)
    assert np.linalg.norm(x - xs) <= 1e-8 * np.linalg.norm(xs)
    # A = identity converges in the first cycle with x = b
    bands = np.zeros((7, 3, 3, 3))
    bands[0] = 1.0
    opI = Operator(3, 3, 3, 0, OFFSETS7, bands)
    xI, repI = gmres(opI, lambda r: r, b, SolverParams(m=5, k_max=0, p1=0))
    assert repI.cycles == 1 and np.allclose(xI, b, rtol=1e-15, atol=1e-15)


def _random_space(op, pc, k, seed):
    U0 = np.random.default_rng(seed).uniform(-1, 1, (op.N, k))
    return refresh_space(lambda v: pc(op.apply(v)), U0)[:2]


def test_rgcrot_cycle_is_optimal_over_U_plus_Krylov():
    """Eqs. (6)-(7): one rGCROT cycle returns the minimiser of
    ||r_hat - A_hat d|| over d in range(U) + K_m(A_C, r0), A_C = (I - C C^T)
    A_hat, r0 = (I - C C^T) r_hat.  Brute force over an explicit basis.
    (The literal Alg. 3 line 13a sign fails this pin -- reading D1.)"""
    prob = channel19(6)
    op, pc, b = _setup(prob)
    U, C = _random_space(op, pc, 4, seed=2)
    m = 5
    prm = SolverParams(m=m, k_max=4, k_t=2, p1=1, tol=1e-30, max_mv=m)
    x, U2, C2, rep = rgcrot(op, pc, b, U.copy(), C.copy(), prm)
    assert rep.cycles == 1
    Ah, _ = _Ahat_dense(op, pc)
    rh = pc(b)
    P = np.eye(op.N) - C @ C.T
    r0 = P @ rh
    K = [r0]
    for _ in range(m - 1):
        K.append(P @ (Ah @ K[-1]))
    Z = np.column_stack([U, _orth(np.column_stack(K))])
    c = np.linalg.lstsq(Ah @ Z, rh, rcond=None)[0]
    xb = Z @ c
    assert np.linalg.norm(x - xb) <= 1e-8 * np.linalg.norm(xb)


@pytest.mark.parametrize("ortho", ["cgs2"])
def test_rgcrot_invariants_every_cycle(ortho):
    """Eq. (4) V _|_ C, eq. (5) A_hat V_m = C B + V_{m+1} H_, Arnoldi
    orthonormality, A_hat U = C and C^T C = I after line 14a,
    residual _|_ C after each cycle (D20), monotone true residual -- for the
    oracle's CGS2 (D8).  (The paper's MGS keeps V orthonormal only to ~2e-12
    here; it is compared in test_rgcrot_mgs_and_cgs2_agree.)"""
    w = get_workload("c2s")
    prob = w.problem()
    op, pc, _ = _setup(prob)
    prm = replace(w.params, ortho=ortho)
    U = np.zeros((op.N, 0))
    C = np.zeros((op.N, 0))
    Anorm = np.abs(to_dense(op)).sum(axis=1).max()
    checks = []

    def hook(d):
        V, H, B = d["V"], d["H"], d["B"]
        m_eff = d["m_eff"]
        Cc, Uc = d["C"], d["U"]
        AV = np.column_stack([pc(op.apply(V[:, j])) for j in range(m_eff)])
        rel5 = np.linalg.norm(AV - Cc @ B - V @ H) / np.linalg.norm(AV)
        orth = np.linalg.norm(V.T @ V - np.eye(V.shape[1]))
        vc = np.linalg.norm(Cc.T @ V) if Cc.shape[1] else 0.0
        checks.append((rel5, orth, vc))

    for t in range(3):
        b = prob.rhs(t).reshape(-1)
        x, U, C, rep = rgcrot(op, pc, b, U, C, prm, hook=hook)
        assert rep.outcome == CONVERGED
        hist = [h[1] for h in rep.history]
        assert all(hist[i + 1] <= hist[i] * (1 + 1e-12) for i in range(len(hist) - 1))
        assert np.linalg.norm(C.T @ C - np.eye(C.shape[1])) <= 1e-12
        AU = np.column_stack([pc(op.apply(U[:, i])) for i in range(U.shape[1])])
        assert np.linalg.norm(AU - C) <= 1e-11 * np.linalg.norm(U)
        assert np.linalg.norm(b - op.apply(x)) <= prm.tol * np.linalg.norm(b)
    for rel5, orth, vc in checks:
        assert rel5 <= 1e-12 and orth <= 1e-12 and vc <= 1e-12


def test_rgcrot_mgs_and_cgs2_agree():
    w = get_workload("c2s")
    prob = w.problem()
    op, pc, b = _setup(prob)
    e = np.zeros((op.N, 0))
    x1, _, _, r1 = rgcrot(op, pc, b, e, e, w.params)
    x2, _, _, r2 = rgcrot(op, pc, b, e, e, replace(w.params, ortho="mgs"))
    assert r1.krylov_mv == r2.krylov_mv
    assert np.linalg.norm(x1 - x2) <= 1e-6 * np.linalg.norm(x1)


def test_rgcrot_solution_vs_direct_solve_c1():
    """BASELINE configs[0] in full: x within kappa*tol of the direct solve."""
    w = get_workload("c1")
    prob = w.problem()
    op, pc, _ = _setup(prob)
    b = prob.rhs(0).reshape(-1)
    e = np.zeros((op.N, 0))
    x, U, C, rep = rgcrot(op, pc, b, e, e, w.params)
    assert rep.outcome == CONVERGED and rep.cycles == 1 and rep.krylov_mv == 20
    D = to_dense(op)
    xs = np.linalg.solve(D, b)
    assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)
    assert np.linalg.norm(b - D @ x) <= 1e-8 * np.linalg.norm(b)


def test_projection_full_space_zero_cycles():
    """r_hat in range(C) -> zero cycles, x = U C^T r_hat (R = I)."""
    prob = convection_diffusion_c1(4)
    op, pc, _ = _setup(prob)
    U, C = _random_space(op, pc, 3, seed=4)
    # b such that M^-1 b = C w: b = M (C w) -- construct via b = A u, u = U w
    wv = np.array([0.3, -1.2, 0.5])
    b = op.apply(U @ wv)
    prm = SolverParams(m=5, k_max=3, k_t=2, tol=1e-8)
    x, _, _, rep = rgcrot(op, pc, b, U, C, prm)
    assert rep.cycles == 0 and rep.krylov_mv == 0 and rep.outcome == CONVERGED
    assert np.linalg.norm(x - U @ wv) <= 1e-10 * np.linalg.norm(U @ wv)


@pytest.mark.parametrize("iters", [1, 3, 6])
def test_bicgstab_matches_scipy(iters):
    """Alg. 2 with right preconditioning == scipy.sparse.linalg.bicgstab
    (same recurrences, r_tilde = r0) after `iters` iterations."""
    prob = porous7(8, 2)
    op, pc, b = _setup(prob)
    prm = SolverParams(tol=1e-30, max_mv=2 * iters)
    x, rep = bicgstab(op, pc, b, prm)
    assert rep.cycles == iters
    A = spla.LinearOperator((op.N, op.N), matvec=op.apply, dtype=np.float64)
    M = spla.LinearOperator((op.N, op.N), matvec=pc, dtype=np.float64)
    xs, info = spla.bicgstab(A, b, x0=np.zeros(op.N), rtol=0.0, atol=0.0, maxiter=iters, M=M)
    assert np.linalg.norm(x - xs) <= 1e-12 * np.linalg.norm(xs)


@pytest.mark.parametrize("iters", [2, 5])
def test_rbicgstab_is_bicgstab_on_projected_operator(iters):
    """Eqs. (8)-(9): rBiCGStab iterates BiCGStab on A_C = (I - C C^T) A with
    r0 = (I - C C^T) b; its pre-line-17a x (= x_final + U xi) equals scipy's
    BiCGStab x on that operator, and line 17a makes b - A x_final equal the
    updated residual (eqs. (10)-(12))."""
    prob = porous7(8, 2)
    op, pc, b = _setup(prob)
    U0 = np.random.default_rng(7).uniform(-1, 1, (op.N, 3))
    U, C, _ = refresh_space(op.apply, U0)
    prm = SolverParams(tol=1e-30, max_mv=2 * iters)
    x, _, _, rep = rbicgstab(op, pc, b, U, C, prm)
    x_pre = x + U @ rep.xi
    P = np.eye(op.N) - C @ C.T
    AC = spla.LinearOperator((op.N, op.N), matvec=lambda v: P @ op.apply(v), dtype=np.float64)
    M = spla.LinearOperator((op.N, op.N), matvec=pc, dtype=np.float64)
    xs, _ = spla.bicgstab(AC, P @ b, x0=np.zeros(op.N), rtol=0.0, atol=0.0, maxiter=iters, M=M)
    assert np.linalg.norm(x_pre - xs) <= 1e-11 * np.linalg.norm(xs)
    assert abs(rep.final_true_res - rep.final_upd_res) <= 1e-10 * np.linalg.norm(b)


def test_rbicgstab_residual_stays_orthogonal_and_certifies():
    """C^T r_i small at every iteration (checked on the final
    updated residual via the certified true residual) and the deferred
    update is exact on a converged run; x matches a direct solve."""
    prob = porous7(10, 2)
    op, pc, b = _setup(prob)
    U0 = np.random.default_rng(9).uniform(-1, 1, (op.N, 4))
    U, C, _ = refresh_space(op.apply, U0)
    prm = SolverParams(tol=1e-10)
    x, _, _, rep = rbicgstab(op, pc, b, U, C, prm)
    assert rep.outcome == CONVERGED
    rt = b - op.apply(x)
    assert np.linalg.norm(C.T @ rt) <= 1e-9 * np.linalg.norm(b)
    xs = np.linalg.solve(to_dense(op), b)
    assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)


def test_bicgstab_forced_breakdown():
    """force a zero denominator.  A = periodic 1-D difference
    (skew-symmetric) with identity preconditioner and b = e_0: r_tilde^T A b
    = 0 exactly -> BREAKDOWN at the first iteration."""
    offs = np.array([(0, 0, 0), (-1, 0, 0), (1, 0, 0)], dtype=np.int8)
    bands = np.zeros((3, 1, 1, 4))
    bands[1] = -1.0
    bands[2] = 1.0
    op = Operator(4, 1, 1, 1, offs, bands)
    b = np.array([1.0, 0, 0, 0])
    x, rep = bicgstab(op, lambda r: r.copy(), b, SolverParams(tol=1e-8))
    assert rep.outcome == BREAKDOWN and rep.cycles == 0
    # nonzero diagonal variant (the one the GPU test uses): A = diag(1,-1,1,1)
    # + skew, b = e0 + e1 -> sigma = b^T A b = 1 - 1 + b^T K b = 0 exactly
    bands[0] = np.array([1.0, -1.0, 1.0, 1.0]).reshape(1, 1, 4)
    op = Operator(4, 1, 1, 1, offs, bands)
    x, rep = bicgstab(op, lambda r: r.copy(), np.array([1.0, 1.0, 0, 0]), SolverParams(tol=1e-8))
    assert rep.outcome == BREAKDOWN and rep.cycles == 0 and rep.krylov_mv == 1


def test_rbicgstab_k0_is_bicgstab_identity_case():
    """A = identity -> first iteration gives x = b (alpha = 1, s = 0)."""
    bands = np.zeros((7, 2, 2, 2))
    bands[0] = 1.0
    op = Operator(2, 2, 2, 0, OFFSETS7, bands)
    b = np.arange(1.0, 9.0)
    x, rep = bicgstab(op, lambda r: r.copy(), b, SolverParams(tol=1e-8))
    assert rep.outcome == CONVERGED and rep.krylov_mv == 1
    assert np.array_equal(x, b)


def test_hybrid_frozen_space_and_conservation():
    """the recycle space handed to every rBiCGStab system after
    the switch is bit-identical; matvec totals add up; the hybrid beats
    plain BiCGStab or is within 20 % on its rBiCGStab phase (reported)."""
    w = get_workload("c3s")
    spaces = []

    def cb(t, tag, x, U, C, rep):
        if tag == "rbicgstab":
            spaces.append((U.copy(), C.copy()))

    out = run_sequence(w, callback=cb)
    tags = [o[0] for o in out]
    assert tags == ["rgcrot"] * 3 + ["rbicgstab"] * (w.n_systems - 3)
    for U, C in spaces[1:]:
        assert np.array_equal(U, spaces[0][0]) and np.array_equal(C, spaces[0][1])
    assert all(o[2].outcome == CONVERGED for o in out)
    U, C = spaces[0]
    prob = w.problem()
    op = Operator.from_problem(prob)
    AU = np.column_stack([op.apply(U[:, i]) for i in range(U.shape[1])])
    assert np.linalg.norm(AU - C) <= 1e-11 * np.linalg.norm(U)   # A U = C (D3)
    assert np.linalg.norm(C.T @ C - np.eye(C.shape[1])) <= 1e-12


def test_recycling_reduces_matvecs_channel():
    """Recycling benefit (S:484 trend): rGCROT beats GMRES(m) on the
    shrunken channel sequence."""
    w = get_workload("c2s")
    rg = sum(o[2].krylov_mv for o in run_sequence(w))
    gm = sum(o[2].krylov_mv for o in run_sequence(w, solver="gmres"))
    assert rg <= 0.8 * gm


def test_gcrot_update_truncation_T1():
    """Line 14a bookkeeping under T1 ("drop the oldest"), checked
    by properties only: k never exceeds k_max; the kept old columns are the
    NEWEST k_t - p ones, untouched and in order; the new C columns lie in
    range(V_{m+1}), have unit norm and are orthogonal to each other; u1 is
    parallel to the cycle correction dx."""
    rng = np.random.default_rng(0)
    N, m, k = 40, 4, 5
    U = rng.standard_normal((N, k))
    C = _orth(rng.standard_normal((N, k)))
    V = _orth(rng.standard_normal((N, m + 1)))
    H = np.triu(rng.standard_normal((m + 1, m)), -1)
    B = rng.standard_normal((k, m))
    y = rng.standard_normal(m)
    dx = rng.standard_normal(N)
    prm = SolverParams(m=m, k_max=5, k_t=3, p1=2)
    U2, C2 = gcrot_update(U, C, V, H, B, y, dx, 1.0, prm)
    assert U2.shape[1] == 3 and C2.shape[1] == 3
    assert np.array_equal(U2[:, 0], U[:, 4]) and np.array_equal(C2[:, 0], C[:, 4])
    Cn = C2[:, 1:]
    assert np.allclose(Cn.T @ Cn, np.eye(2), atol=1e-14)
    assert np.linalg.norm(Cn - V @ (V.T @ Cn)) <= 1e-14
    cos = abs(U2[:, 1] @ dx) / (np.linalg.norm(U2[:, 1]) * np.linalg.norm(dx))
    assert abs(cos - 1.0) <= 1e-14
    # without truncation (k_max large) every old column is kept
    U3, C3 = gcrot_update(U, C, V, H, B, y, dx, 1.0, replace(prm, k_max=10, k_t=8))
    assert U3.shape[1] == k + 2 and np.array_equal(U3[:, :k], U)


def test_refresh_space_drops_dependent_column():
    """Line 1a's rank-drop branch: when op(U) is rank deficient
    (U's third column is a combination of the first two), the first column
    whose QR pivot vanishes is dropped; the result still satisfies
    op(U) = C, C^T C = I, and range(C) equals the column space of the
    original op(U) (projectors compared against an SVD basis)."""
    prob = convection_diffusion_c1(4)
    op, pc, _ = _setup(prob)
    rng = np.random.default_rng(3)
    U0 = rng.standard_normal((op.N, 4))
    U0[:, 2] = 0.5 * U0[:, 0] - 2.0 * U0[:, 1]
    ahat = lambda v: pc(op.apply(v))
    U, C, apps = refresh_space(ahat, U0.copy())
    assert U.shape[1] == 3 and C.shape[1] == 3 and apps == 4 + 3
    assert np.linalg.norm(C.T @ C - np.eye(3)) <= 1e-13
    AU = np.column_stack([ahat(U[:, i]) for i in range(3)])
    assert np.linalg.norm(AU - C) <= 1e-11 * np.linalg.norm(U)
    AU0 = np.column_stack([ahat(U0[:, i]) for i in range(4)])
    Us, sv, _ = np.linalg.svd(AU0, full_matrices=False)
    assert sv[3] <= 1e-12 * sv[0]
    P1 = Us[:, :3] @ Us[:, :3].T
    assert np.linalg.norm(C @ C.T - P1) <= 1e-10
    # the dropped column is the dependent one (index 2): columns 0, 1, 3 span U
    Ukeep = U0[:, [0, 1, 3]]
    coef = np.linalg.lstsq(Ukeep, U, rcond=None)[0]
    assert np.linalg.norm(Ukeep @ coef - U) <= 1e-10 * np.linalg.norm(U)


@pytest.mark.parametrize("p1", [1, 2])
def test_gcrot_update_columns_from_the_cycle(p1):
    """Line 14a (reading D11) against what one rGCROT cycle fixes, not
    against its own formulas: the cycle's correction minimises the residual
    over range(U) + K_m (eqs. (6)-(7)), so the post-cycle preconditioned
    residual is orthogonal to A_hat of the whole search space.  Every column
    the update adds comes from that space (c1 = A_hat u1 with u1 the
    normalised correction; c2 = A_hat u2, u2 in span(V_j*, U)), hence
    C_new^T r_new = 0; u1 is parallel to the cycle's correction itself (x
    minus line 1b's projection U C^T r_hat0, x0 = 0); A_hat U = C and
    C^T C = I.  A new column taken from the Krylov
    basis itself (V rather than V_{m+1} h) or from the uncorrected x would
    fail the first two checks."""
    prob = channel19(6)
    op, pc, b = _setup(prob)
    U, C = _random_space(op, pc, 3, seed=5)
    m = 5
    prm = SolverParams(m=m, k_max=6, k_t=4, p1=p1, tol=1e-30, max_mv=m)
    x, U2, C2, rep = rgcrot(op, pc, b, U.copy(), C.copy(), prm)
    assert rep.cycles == 1 and U2.shape[1] == 3 + p1
    rn = pc(b - op.apply(x))
    assert np.linalg.norm(C2.T @ rn) <= 1e-10 * np.linalg.norm(rn)
    # the cycle's own correction: x minus line 1b's projection U C^T r_hat0
    dx = x - U @ (C.T @ pc(b))
    u1 = U2[:, 3]
    cos = abs(u1 @ dx) / (np.linalg.norm(u1) * np.linalg.norm(dx))
    assert abs(cos - 1.0) <= 1e-12
    AU = np.column_stack([pc(op.apply(U2[:, i])) for i in range(U2.shape[1])])
    assert np.linalg.norm(AU - C2) <= 1e-11 * np.linalg.norm(U2)
    assert np.linalg.norm(C2.T @ C2 - np.eye(C2.shape[1])) <= 1e-12
    # the old columns are kept as they were (no truncation at k = 3 + p1 <= k_max)
    assert np.array_equal(U2[:, :3], U) and np.array_equal(C2[:, :3], C)


def test_t2_directions_are_principal_vectors():
    """T2 (reading R13): the kept directions C W are the principal vectors
    of range(C) w.r.t. the cycle's image space [C V_{m+1}] [B; H_]
    (eq. (5)).  Pinned against scipy.linalg.subspace_angles (an
    independent principal-angle routine): the cosines of the angles of
    each kept direction to the image equal the `keep` largest cosines of
    the principal angles, in order; W has orthonormal columns and the
    sign rule holds."""
    import scipy.linalg as sla
    from oracle.krylov import t2_directions
    rng = np.random.default_rng(4)
    N, m, k, keep = 60, 6, 8, 5
    CV = _orth(rng.standard_normal((N, k + m + 1)))
    C, V = CV[:, :k], CV[:, k:]
    H = np.triu(rng.standard_normal((m + 1, m)), -1)
    B = rng.standard_normal((k, m))
    W = t2_directions(B, H, keep)
    assert np.allclose(W.T @ W, np.eye(keep), atol=1e-13)
    img = _orth(CV @ np.vstack([B, H]))
    cos_ref = np.sort(np.cos(sla.subspace_angles(C, img)))[::-1][:keep]
    cos_kept = np.linalg.norm(img.T @ (C @ W), axis=0)
    assert np.allclose(cos_kept, cos_ref, atol=1e-12)
    for j in range(keep):
        assert W[np.argmax(np.abs(W[:, j])), j] > 0


def test_rgcrot_T2_invariants_and_solution():
    """rGCROT with T2 truncation keeps A_hat U = C, C^T C = I and solves
    the shrunken channel sequence to tol (the invariants of S:275-282)."""
    w = get_workload("c2s")
    prob = w.problem()
    op, pc, _ = _setup(prob)
    prm = replace(w.params, trunc="T2")
    U = np.zeros((op.N, 0))
    C = np.zeros((op.N, 0))
    truncated = 0
    for t in range(4):
        b = prob.rhs(t).reshape(-1)
        k_before = U.shape[1]
        x, U, C, rep = rgcrot(op, pc, b, U, C, prm)
        truncated += rep.cycles > 0 and k_before + rep.cycles * prm.p1 > prm.k_max
        assert rep.outcome == CONVERGED
        assert U.shape[1] <= prm.k_max
        assert np.linalg.norm(C.T @ C - np.eye(C.shape[1])) <= 1e-12
        AU = np.column_stack([pc(op.apply(U[:, i])) for i in range(U.shape[1])])
        assert np.linalg.norm(AU - C) <= 1e-11 * np.linalg.norm(U)
        assert np.linalg.norm(b - op.apply(x)) <= prm.tol * np.linalg.norm(b)
    assert truncated


def _with(w0, **kw):
    from problems.workloads import Workload
    return Workload(w0.name, w0.make_problem, replace(w0.params, **kw), w0.n_systems,
                    w0.epoch_every, w0.description)


def test_hybrid_switchback_policy():
    """P:668-669 / SPEC hybrid allow_switchback (reading R16): an rBiCGStab
    solve that does not converge is re-solved by rGCROT from x = 0 and the
    run continues with rBiCGStab.  Instability threshold 0.15 ||r0|| makes
    exactly system 5 of c3s unstable (its residual peaks at 0.26 ||r0||, the
    others stay below 0.095 ||r0||); counts are conserved."""
    from oracle.krylov import OUTCOME_NAMES
    w = _with(get_workload("c3s"), divergence=0.15)
    plain = run_sequence(w)
    assert [OUTCOME_NAMES[r.outcome] for _, _, r in plain][5] == "UNSTABLE"
    out = run_sequence(w, switchback=True)
    tags = [t for t, _, _ in out]
    assert tags == ["rgcrot"] * 3 + ["rbicgstab", "rbicgstab", "rbicgstab+rgcrot", "rbicgstab", "rbicgstab"]
    assert all(rep.outcome == CONVERGED for _, _, rep in out)
    rep5 = out[5][2]
    failed = plain[5][2].krylov_mv
    assert rep5.krylov_mv > failed and rep5.cycles >= 1


def test_hybrid_refresh_on_epoch_policy():
    """P:666-667 "intermittent solves with rGCROT to update the recycle space
    ... when the system matrix changes" (R16): with A epochs every 3 systems
    and the switch after 3, systems 3 and 6 (first of a new epoch) are solved
    by rGCROT, the others by rBiCGStab; every system converges.  With
    refresh_every = 2 every second post-switch system is an rGCROT solve."""
    w = get_workload("c4hs")
    out = run_sequence(w, refresh_on_epoch=True)
    assert [t for t, _, _ in out] == ["rgcrot"] * 4 + ["rbicgstab"] * 2 + ["rgcrot"] + ["rbicgstab"] * 2
    assert all(r.outcome == CONVERGED for _, _, r in out)
    every = run_sequence(w, refresh_every=2)
    assert [t for t, _, _ in every] == ["rgcrot"] * 3 + ["rbicgstab", "rgcrot"] * 3


def test_cgs2g_equals_cgs2_coefficients():
    """R19: the Gram-corrected coefficients (2I - G) Q^T w equal CGS2's
    g1 + g2 = Q^T w + Q^T (w - Q Q^T w) in exact arithmetic; on a basis whose
    orthogonality is perturbed at 1e-9 they agree to O(1e-17) relative
    (second order in the perturbation), and both leave w orthogonal to Q."""
    rng = np.random.default_rng(6)
    N, n = 400, 12
    Q = _orth(rng.standard_normal((N, n)))
    Q = Q + 1e-9 * rng.standard_normal((N, n))
    w = rng.standard_normal(N)
    g1 = Q.T @ w
    g2 = Q.T @ (w - Q @ g1)
    h = 2.0 * g1 - (Q.T @ Q) @ g1
    assert np.linalg.norm(h - (g1 + g2)) <= 1e-15 * np.linalg.norm(g1)
    wg = w - Q @ h
    assert np.linalg.norm(Q.T @ wg) <= 1e-14 * np.linalg.norm(w)
