"""Pins for oracle/kernels.py (the per-kernel references) against exact
rational arithmetic, algebraic identities and the pinned solver oracle
(oracle.krylov.rbicgstab, itself pinned to scipy's BiCGStab)."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import kernels as K
from oracle.krylov import refresh_space, rbicgstab
from oracle.stencil import Operator
from problems import SolverParams
from problems.stencils import porous7


def _rand(n, ncol, seed):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1, 1, n) for _ in range(ncol)], rng.uniform(-1, 1, n)


def _exact_dot(a, b):
    return float(sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b)))


def test_block_dot_exact_rational():
    Q, w = _rand(11, 5, 0)
    got = K.block_dot(Q, w)
    for c in range(5):
        ref = _exact_dot(Q[c], w)
        scale = float(np.abs(Q[c]) @ np.abs(w))
        assert abs(got[c] - ref) <= 1e-16 * scale


def test_block_update_and_dots_exact_rational():
    Q, w = _rand(9, 4, 1)
    g = np.random.default_rng(2).uniform(-1, 1, 4)
    d = np.random.default_rng(3).uniform(-1, 1, 9)
    wn, (dd, nn) = K.block_update(Q, g, w, (d, None))
    for i in range(9):
        ex = Fraction(float(w[i])) - sum(Fraction(float(g[c])) * Fraction(float(Q[c][i])) for c in range(4))
        assert abs(wn[i] - float(ex)) <= 4e-16 * (abs(w[i]) + sum(abs(g[c] * Q[c][i]) for c in range(4)))
    assert abs(dd - _exact_dot(wn, d)) <= 1e-15 * float(np.abs(wn) @ np.abs(d))
    assert abs(nn - _exact_dot(wn, wn)) <= 1e-15 * nn


def test_block_project_is_orthogonal_projector():
    """eq. (8): (I - C C^T) w is orthogonal to range(C) for orthonormal C,
    and w = w_new + C eta."""
    rng = np.random.default_rng(4)
    C, _ = np.linalg.qr(rng.uniform(-1, 1, (200, 7)))
    Q = [C[:, c].copy() for c in range(7)]
    w = rng.uniform(-1, 1, 200)
    eta, wn, nn = K.block_project(Q, w)
    assert np.max(np.abs(C.T @ wn)) <= 1e-14 * np.linalg.norm(w)
    assert np.max(np.abs(wn + C @ eta - w)) <= 1e-14 * np.linalg.norm(w)
    assert abs(nn - wn @ wn) <= 1e-14 * nn
    assert np.allclose(eta, C.T @ w, rtol=0, atol=1e-14)


def test_gram_update_equals_two_cgs_passes_exact():
    """R19's algebra: with G the exact Gram matrix of Q, h = 2g - Gg equals
    the two classical Gram-Schmidt passes' coefficients g1 + Q^T (w - Q g1)
    (evaluated here in exact rational arithmetic, independently of
    gram_matrix / gram_update)."""
    n, ncol, k = 10, 5, 2
    rng = np.random.default_rng(5)
    Cq, _ = np.linalg.qr(rng.uniform(-1, 1, (n, k)))
    V = rng.uniform(-1, 1, (n, ncol - k))
    Qm = np.column_stack([Cq, V])
    Q = [Qm[:, c].copy() for c in range(ncol)]
    w = rng.uniform(-1, 1, n)
    Fq = [[Fraction(float(x)) for x in q] for q in Q]
    Fw = [Fraction(float(x)) for x in w]
    fdot = lambda a, b: sum(x * y for x, y in zip(a, b))
    g1 = [fdot(q, Fw) for q in Fq]
    w1 = [Fw[i] - sum(g1[c] * Fq[c][i] for c in range(ncol)) for i in range(n)]
    g2 = [fdot(q, w1) for q in Fq]
    h_exact = [float(a + b) for a, b in zip(g1, g2)]
    # grow rows i >= k: exact q_i^T q_l; C block taken as I (C^T C = I to rounding)
    grow = [[float(fdot(Fq[i], Fq[l])) if i >= k else 0.0 for l in range(ncol)] for i in range(ncol)]
    g = np.array([float(x) for x in g1])
    h, wn, nn = K.gram_update(Q, k, g, grow, w)
    scale = np.linalg.norm(w) * max(1.0, np.abs(Qm).sum(axis=0).max())
    assert np.max(np.abs(h - np.array(h_exact))) <= 1e-13 * scale
    w2 = w - Qm @ h
    assert np.max(np.abs(wn - w2)) <= 1e-13 * scale


def test_gram_update_with_identity_gram_is_block_update():
    Q, w = _rand(50, 6, 6)
    g = np.array(K.block_dot(Q, w))
    grow = [[1.0 if i == l else 0.0 for l in range(6)] for i in range(6)]
    h, wn, _ = K.gram_update(Q, 6, g, grow, w)
    assert np.array_equal(h, g)                      # 2g - I g, exact
    ref, _ = K.block_update(Q, g, w)
    assert np.max(np.abs(wn - ref)) == 0.0


def test_normalize_and_breakdown():
    w = np.random.default_rng(7).uniform(-1, 1, 30)
    v, f = K.normalize(w, float(w @ w), 1.0)
    assert f == 0.0 and abs(np.linalg.norm(v) - 1.0) <= 1e-15
    v, f = K.normalize(1e-20 * w, float((1e-20 * w) @ (1e-20 * w)), 1.0)
    assert f == 1.0 and not v.any()


def test_lincomb_and_rotate_exact_rational():
    Q, _ = _rand(8, 4, 8)
    rng = np.random.default_rng(9)
    coef = rng.uniform(-1, 1, (2, 4))
    outs = [rng.uniform(-1, 1, 8), rng.uniform(-1, 1, 8)]
    res = K.lincomb(Q, coef, outs, [0.5, -2.0], [False, True])
    for o, (sc, acc) in enumerate(((0.5, False), (-2.0, True))):
        for i in range(8):
            ex = Fraction(sc) * sum(Fraction(float(coef[o][c])) * Fraction(float(Q[c][i])) for c in range(4))
            if acc:
                ex += Fraction(float(outs[o][i]))
            assert abs(res[o][i] - float(ex)) <= 1e-15 * (4 + abs(outs[o][i]))
    T = rng.uniform(-1, 1, (4, 4))
    rot = K.rotate(Q, T, kout=3)
    assert len(rot) == 3
    for c in range(3):
        for i in range(8):
            ex = sum(Fraction(float(T[l][c])) * Fraction(float(Q[l][i])) for l in range(4))
            assert abs(rot[c][i] - float(ex)) <= 1e-15 * 4


def test_bicg_xr_modes():
    """Lines 10-10a (exact exit) and the D17 breakdown guards."""
    rng = np.random.default_rng(10)
    x, r, s, t, ph, sh, rt = (rng.uniform(-1, 1, 6) for _ in range(7))
    base = dict(rho=0.3, sigma=0.5, ss=1.0, ts=0.2, tt=0.4)
    m, xn, rn, _, _, _ = K.bicg_xr(x, r, s, t, ph, sh, rt, base)
    assert m == 0 and np.allclose(xn, x + 0.6 * ph + 0.5 * sh, rtol=0, atol=1e-15)
    assert np.allclose(rn, s - 0.5 * t, rtol=0, atol=1e-15)
    m, xn, rn, _, _, _ = K.bicg_xr(x, r, s, t, ph, sh, rt, dict(base, ss=0.0))
    assert m == 1 and np.array_equal(rn, s) and np.allclose(xn, x + 0.6 * ph, rtol=0, atol=1e-15)
    for bad in (dict(base, sigma=0.0), dict(base, tt=0.0), dict(base, ts=0.0)):
        m, xn, rn, _, _, _ = K.bicg_xr(x, r, s, t, ph, sh, rt, bad)
        assert m == 2 and np.array_equal(xn, x) and np.array_equal(rn, r)


@pytest.mark.parametrize("k", [0, 3])
def test_bicg_kernels_compose_to_rbicgstab(k):
    """bicg_p -> A -> bicg_project_s -> A -> block_dot / block_update ->
    bicg_xr, iterated, reproduces oracle.krylov.rbicgstab's per-iteration
    scalars and iterates (one-sweep Jacobi M^-1 = w_l D^-1, so the fused
    first sweep is the whole preconditioner)."""
    prob = porous7(8, 2)
    op = Operator.from_problem(prob)
    b = prob.rhs(1).reshape(-1)
    wl = 0.8
    invD = 1.0 / op.diag()
    pc = lambda r: (wl * r) * invD
    U = np.zeros((op.N, 0))
    C = np.zeros((op.N, 0))
    if k:
        U, C, _ = refresh_space(op.apply, np.random.default_rng(11).uniform(-1, 1, (op.N, k)))
    iters = 6
    hooks = []
    prm = SolverParams(tol=1e-30, max_mv=2 * iters)
    rbicgstab(op, pc, b, U, C, prm, hook=hooks.append)
    assert len(hooks) == iters
    Q = [C[:, c].copy() for c in range(k)]
    bnorm = np.linalg.norm(b)
    if k:
        eta0, r, _ = K.block_project(Q, b)
        xi = -eta0
    else:
        r, xi = b.copy(), None
    rt = r.copy()
    x = np.zeros(op.N)
    p = v = None
    cur = dict(rho=K._dot(rt, r), rr=K._dot(r, r))
    prev = None
    r0n = np.sqrt(cur["rr"])
    for i in range(iters):
        stop, p, ph = K.bicg_p(i == 0, r, p, v, invD, wl, cur, prev, 1e-30 * bnorm, 1e4 * r0n)
        assert not stop
        v = op.apply(ph)
        if k:
            eta1, v, sigma, s, sh, ss = K.bicg_project_s(Q, v, rt, r, invD, wl, cur["rho"])
        else:
            eta1 = None
            sigma = K._dot(rt, v)
            s, sh, ss = K.bicg_s(r, v, invD, wl, cur["rho"], sigma)
        t = op.apply(sh)
        if k:
            eta2 = K.block_dot(Q, t)
            t, (ts, tt) = K.block_update(Q, eta2, t, (s, None))
        else:
            eta2 = None
            ts, tt = K._dot(t, s), K._dot(t, t)
        cur.update(sigma=sigma, ss=ss, ts=ts, tt=tt, flag=0.0)
        mode, x, r, xi, rho_n, rr_n = K.bicg_xr(x, r, s, t, ph, sh, rt, cur, xi, eta1, eta2)
        assert mode == 0
        h = hooks[i]
        for key in ("rho", "sigma", "ss", "ts", "tt"):
            assert abs(cur[key] - h[key]) <= 1e-12 * abs(h[key]), (i, key)
        assert abs(rr_n - h["rr"]) <= 1e-12 * h["rr"]
        assert np.linalg.norm(x - h["x"]) <= 1e-12 * np.linalg.norm(h["x"])
        if k:
            assert np.linalg.norm(xi - h["xi"]) <= 1e-12 * np.linalg.norm(h["xi"])
        prev = dict(cur)
        cur = dict(rho=rho_n, rr=rr_n)


def test_project_update_exact_rational():
    C, r = _rand(7, 3, 12)
    U, x = _rand(7, 3, 13)
    xi = np.random.default_rng(14).uniform(-1, 1, 3)
    rn, xn, nn = K.project_update(C, U, xi, r, x)
    for i in range(7):
        er = Fraction(float(r[i])) - sum(Fraction(float(xi[c])) * Fraction(float(C[c][i])) for c in range(3))
        ex = Fraction(float(x[i])) + sum(Fraction(float(xi[c])) * Fraction(float(U[c][i])) for c in range(3))
        assert abs(rn[i] - float(er)) <= 1e-15 * 4 and abs(xn[i] - float(ex)) <= 1e-15 * 4
    assert abs(nn - _exact_dot(rn, rn)) <= 1e-15 * nn
    rn2, xn2, _ = K.project_update(C, U, xi, r)
    assert xn2 is None and np.array_equal(rn2, rn)
