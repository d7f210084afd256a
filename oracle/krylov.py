"""Oracle O3-O7: rGCROT(m,k), GMRES(m), rBiCGStab, BiCGStab and the
hybrid sequence driver, step by step in the paper's order and notation.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings of the paper are
marked [Dn] where they are applied.  Notation: A the operator, M^-1 the
Jacobi(5+1) map, A_hat = M^-1 A (left preconditioning for GMRES/rGCROT,
P:148), (U, C) the recycle space with A_hat U = C (rGCROT) or A U = C
(rBiCGStab), R absorbed into U after every QR so R = I [D14].

Pins (tests/oracle/): rGCROT's cycle iterate equals the brute-force
minimiser of ||r_hat - A_hat d|| over d in range(U) + K_m(A_C, r0)
(eqs. (6)-(7)); GMRES(m) equals the brute-force minimal
residual over the explicit Krylov space (Alg. 1 l.12); k = 0 reduces
rGCROT to GMRES(m) and rBiCGStab to BiCGStab; BiCGStab
iterates equal scipy.sparse.linalg.bicgstab's; rBiCGStab's pre-17a
iterates equal scipy's BiCGStab run on A_C = (I - C C^T) A (eq. (8)-(9));
invariants C^T C = I, A_hat U = C, V _|_ C, eq. (5); dense direct solves.
The line-14a update is pinned by what one cycle fixes (every added
column from the cycle's search space: the post-cycle residual is
orthogonal to all of C; u1 parallel to the cycle's correction; the
invariants above).

PARITY UNPINNED: the choice of the p1 = 2 candidate (j* = argmax |y_j|
over j <= floor(m/2), reading D11) -- the paper gives no algorithm for
line 14a, so nothing outside this oracle fixes which second
column is added; only its properties (taken from the cycle's search
space, A_hat U = C, C^T C = I) are pinned.

Orthogonalisation (D8): `cgs2` (block classical Gram-Schmidt over
[C V_j] applied twice, the default) or `mgs` (the literal loops of Alg. 3
lines 6a-9).  librk's Gram-corrected CGS2 (R19) is NOT
implemented here: the oracle stays the textbook scheme, and the GPU's
one-update variant is checked against it.
"""
from dataclasses import dataclass, field

import numpy as np

CONVERGED, MAX_MATVECS, BREAKDOWN, STAGNATION, UNSTABLE, DRIFT = range(6)
OUTCOME_NAMES = ["CONVERGED", "MAX_MATVECS", "BREAKDOWN", "STAGNATION", "UNSTABLE", "DRIFT"]


@dataclass
class Report:
    outcome: int = MAX_MATVECS
    krylov_mv: int = 0          # applications of the (preconditioned) operator in the Krylov loop
    op_apps: int = 0            # other applications of A (true residuals, refresh, certification)
    cycles: int = 0             # rGCROT cycles or rBiCGStab iterations
    bnorm: float = 0.0
    final_true_res: float = float("nan")
    final_upd_res: float = float("nan")
    history: list = field(default_factory=list)   # (krylov_mv, ||b - A x||, preconditioned/updated ||r||)
    k_after: int = 0
    xi: object = None           # rBiCGStab: the deferred U-coefficients applied at line 17a


def _norm(v):
    return float(np.sqrt(np.dot(v, v)))


# ------------------------------------------------------------------ line 1a
def refresh_space(apply_op, U):
    """Alg. 3 line 1a / Alg. 4 line 1b: C~ = op(U); C~ = C R (thin QR,
    diag(R) > 0 [D15]); U <- U R^-1 so that op(U) = C with R = I [D14].
    A column whose pivot |R_ii| <= 1e-12 max|R_jj| is dropped (first such
    column, then QR again).  Returns (U, C, applications)."""
    apps = 0
    while U.shape[1] > 0:
        Ct = np.column_stack([apply_op(U[:, i]) for i in range(U.shape[1])])
        apps += U.shape[1]
        Q, R = np.linalg.qr(Ct)
        s = np.sign(np.diag(R))
        s[s == 0] = 1.0
        Q = Q * s
        R = (R.T * s).T
        dg = np.abs(np.diag(R))
        bad = np.nonzero(dg <= 1e-12 * dg.max())[0]
        if bad.size:
            U = np.delete(U, bad[0], axis=1)
            continue
        U = np.linalg.solve(R.T, U.T).T        # U R^-1
        return U, Q, apps
    return U, np.zeros_like(U), apps


# ----------------------------------------------------------------- line 14a
def gcrot_update(U, C, V, H, B, y, dx, rho, prm):
    """Alg. 3 line 14a "Update U and C if desired" -- reading
    [D11].  Pinned by test_gcrot_update_columns_from_the_cycle (added
    columns from the cycle's search space, u1 parallel to the correction,
    A_hat U = C, C^T C = I) and test_gcrot_update_truncation_T1; the p1 = 2
    candidate choice is the reading's, not the paper's.

    Extension by the normalised cycle correction: with zeta = H_ y and
    gamma = ||zeta||, u1 = dx/gamma and c1 = V_{m+1} zeta/gamma, so that
    A_hat u1 = c1 exactly by eq. (5) (no matvec).  For p1 = 2 a second
    candidate from the pool j <= floor(m/2): j* = argmax |y_j| (ties to the
    smaller j), h* = H_(:, j*), u = v_j* - U B(:, j*) satisfies
    A_hat u = V_{m+1} h*; it is orthogonalised against c1 in coefficient
    space.  Truncation T1: if k + p > k_max keep the newest k_t - p old
    columns (drop the oldest); T2 (prm.trunc == "T2"): keep the
    k_t - p directions of range(C) with the smallest principal angles to the
    cycle's image space (t2_directions).  Columns are ordered oldest first."""
    m_eff = len(y)
    k = U.shape[1]
    zeta = H @ y
    gamma = _norm(zeta)
    newU, newC = [], []
    if gamma > 1e-14 * rho and prm.p1 >= 1:
        zh = zeta / gamma
        u1 = dx / gamma
        c1 = V @ zh
        newU.append(u1)
        newC.append(c1)
        if prm.p1 >= 2:
            pool = max(1, m_eff // 2)
            js = int(np.argmax(np.abs(y[:pool])))
            hs = H[:, js]
            s = float(zh @ hs)
            cp = hs - zh * s
            delta = _norm(cp)
            if delta > 1e-12 * _norm(hs):
                u2 = (V[:, js] - U @ B[:, js] - u1 * s) / delta
                c2 = V @ (cp / delta)
                newU.append(u2)
                newC.append(c2)
    p = len(newU)
    if p == 0:
        return U, C
    if k + p > prm.k_max:
        keep = max(0, prm.k_t - p)
        if getattr(prm, "trunc", "T1") == "T2" and 0 < keep <= min(k, m_eff):
            W = t2_directions(B, H, keep)
            U = U @ W
            C = C @ W
        else:
            U = U[:, k - keep:]
            C = C[:, k - keep:]
    U = np.column_stack([U] + newU)
    C = np.column_stack([C] + newC)
    return U, C


def t2_directions(B, H, keep):
    """Truncation T2 (the GCROT angle criterion the
    paper names at P:462-463): the cycle's image space is
    A_hat V_m = [C V_{m+1}] [B; H_] (eq. (5)); with Q = qr([B; H_]) the
    cosines of the principal angles between range(C) and that image are the
    singular values of Q(1:k, :) = W S Z^T.  Keep the `keep` directions of
    range(C) closest to the image (largest singular values): U <- U W,
    C <- C W with W = W[:, :keep], each column sign-normalised so that its
    largest-|.| entry is positive.  C W stays orthonormal and A_hat U W = C W.
    Used when keep <= min(k, m_eff) (reading R13), else T1."""
    k = B.shape[0]
    Q, _ = np.linalg.qr(np.vstack([B, H]))
    W, _, _ = np.linalg.svd(Q[:k, :])
    W = W[:, :keep].copy()
    for j in range(keep):
        i = int(np.argmax(np.abs(W[:, j])))
        if W[i, j] < 0:
            W[:, j] = -W[:, j]
    return W


# --------------------------------------------------------------- O3 rGCROT
def rgcrot(op, pc, b, U, C, prm, valid=True, hook=None):
    """Alg. 3 rGCROT(m,k), left preconditioned (A_hat = M^-1 A).

    Returns (x, U, C, report).  x_hat = 0.  Convergence is the
    true residual ||b - A x|| <= tol ||b|| tested at cycle end [D4, D5].
    hook(dict) is called at every cycle end with the cycle's quantities
    (tests inspect eq. (4)/(5) there)."""
    N = b.size
    rep = Report(bnorm=_norm(b))
    x = np.zeros(N)
    if rep.bnorm == 0.0:
        rep.outcome, rep.final_true_res, rep.k_after = CONVERGED, 0.0, U.shape[1]
        return x, U, C, rep
    tol, m = prm.tol, prm.m

    def ahat(v):
        return pc(op.apply(v))

    # line 1a: refresh when U was set without C or A changed
    if U.shape[1] > 0 and not valid:
        U, C, apps = refresh_space(ahat, U)
        rep.op_apps += apps
    # line 1: r_hat = M^-1 (b - A x_hat) = M^-1 b
    r_hat = pc(b)
    # line 1b: xi = C^T r_hat; r0 = r_hat - C xi; x0 = x_hat + U xi  (R = I)
    xi = C.T @ r_hat
    r = r_hat - C @ xi
    x = x + U @ xi
    # [D6] zero-cycle exit
    if _norm(r) <= tol * _norm(r_hat):
        rt = b - op.apply(x)
        rep.op_apps += 1
        if _norm(rt) <= tol * rep.bnorm:
            rep.outcome = CONVERGED
            rep.final_true_res = _norm(rt)
            rep.final_upd_res = _norm(r)
            rep.k_after = U.shape[1]
            return x, U, C, rep
    cycle = 0
    while rep.krylov_mv < prm.max_mv:
        if cycle > 0:
            # [D20] re-project the recomputed residual against C
            xi = C.T @ r
            r = r - C @ xi
            x = x + U @ xi
        k = U.shape[1]
        rho = _norm(r)                                     # rho_i
        V = np.zeros((N, m + 1))
        H = np.zeros((m + 1, m))
        Bm = np.zeros((k, m))
        V[:, 0] = r / rho                                  # line 4
        m_eff = m
        for j in range(m):                                 # line 5
            w = ahat(V[:, j])                              # line 6
            rep.krylov_mv += 1
            w_in = _norm(w)
            if prm.ortho == "mgs":
                for l in range(k):                         # lines 6a-6c
                    Bm[l, j] = C[:, l] @ w
                    w = w - C[:, l] * Bm[l, j]
                for l in range(j + 1):                     # lines 7-9
                    H[l, j] = V[:, l] @ w
                    w = w - V[:, l] * H[l, j]
            else:
                # [D8] block classical Gram-Schmidt over [C V_j], applied twice
                Q = np.column_stack([C, V[:, :j + 1]])
                for _ in range(2):
                    g = Q.T @ w
                    w = w - Q @ g
                    Bm[:, j] += g[:k]
                    H[:j + 1, j] += g[k:]
            H[j + 1, j] = _norm(w)                          # line 10
            if H[j + 1, j] <= 1e-14 * w_in:                 # [D18] happy breakdown
                m_eff = j + 1
                break
            V[:, j + 1] = w / H[j + 1, j]
        Hm = H[:m_eff + 1, :m_eff]
        e1 = np.zeros(m_eff + 1)
        e1[0] = rho
        y = np.linalg.lstsq(Hm, e1, rcond=None)[0]         # line 12
        z = -(Bm[:, :m_eff] @ y)                           # line 12a
        dx = V[:, :m_eff] @ y + U @ z                      # lines 13-13a per eq. (6) [D1]
        x = x + dx
        rt = b - op.apply(x)                               # line 14
        rep.op_apps += 1
        true_res = _norm(rt)
        prec_res = _norm(e1 - Hm @ y)
        rep.history.append((rep.krylov_mv, true_res, prec_res))
        if hook is not None:
            hook(dict(U=U, C=C, V=V[:, :m_eff + 1], H=Hm, B=Bm[:, :m_eff], y=y, dx=dx,
                      rho=rho, x=x, m_eff=m_eff))
        U, C = gcrot_update(U, C, V[:, :m_eff + 1], Hm, Bm[:, :m_eff], y, dx, rho, prm)  # 14a [D21]
        cycle += 1
        rep.cycles = cycle
        rep.final_true_res = true_res
        rep.final_upd_res = prec_res
        if true_res <= tol * rep.bnorm:
            rep.outcome = CONVERGED
            break
        r = pc(rt)
    else:
        rep.outcome = MAX_MATVECS
    rep.k_after = U.shape[1]
    return x, U, C, rep


def gmres(op, pc, b, prm):
    """Alg. 1 GMRES(m) = rGCROT with an empty recycle space and no update
    ("The changes from the GMRES(m) algorithm are ...")."""
    from dataclasses import replace
    N = b.size
    e = np.zeros((N, 0))
    x, _, _, rep = rgcrot(op, pc, b, e, e, replace(prm, p1=0, k_max=0))
    return x, rep


# ------------------------------------------------------------ O5 rBiCGStab
def rbicgstab(op, pc, b, U, C, prm, valid=True, x_hat=None, hook=None):
    """Alg. 4 rBiCGStab with one recycle space, right preconditioned
    (P:148 [D2]): the iterated operator is A_C M^-1 with A_C = (I - C C^T) A
    (eq. (8)); x-updates use p_hat = M^-1 p, s_hat = M^-1 s [D22]; U-updates
    deferred in xi and applied once at line 17a.
    Returns (x, U, C, report); (U, C) are frozen (only refreshed if invalid).
    hook(dict) is called after every completed iteration with its scalars
    (rho, sigma, ||s||^2, t^T s, t^T t, ||r_{i+1}||^2; tests compare them)."""
    N = b.size
    rep = Report(bnorm=_norm(b))
    tol = prm.tol
    if rep.bnorm == 0.0:
        rep.outcome, rep.final_true_res, rep.k_after = CONVERGED, 0.0, U.shape[1]
        return np.zeros(N), U, C, rep
    if U.shape[1] > 0 and not valid:                       # line 1b [D3]: C R = qr(A U)
        U, C, apps = refresh_space(op.apply, U)
        rep.op_apps += apps
    x = np.zeros(N) if x_hat is None else x_hat.copy()
    while True:
        r = b - op.apply(x) if x.any() else b.copy()       # line 1: r_hat = b - A x_hat
        if x.any():
            rep.op_apps += 1
        eta = C.T @ r                                      # line 1c
        r = r - C @ eta
        xi = -eta
        rt = r.copy()                                      # r_tilde = r0 [D16]
        r0n = _norm(r)
        i = 0
        rho_old = alpha = omega = 1.0
        p = v = None
        status = None
        while _norm(r) > tol * rep.bnorm and rep.krylov_mv < prm.max_mv:   # line 3
            rho = float(rt @ r)                            # line 4
            if rho == 0.0:                                 # line 5
                status = BREAKDOWN
                break
            if i == 0:                                     # line 6
                p = r.copy()
            else:
                beta = (rho / rho_old) * (alpha / omega)
                p = r + beta * (p - omega * v)
            ph = pc(p)                                     # right preconditioning
            v = op.apply(ph)                               # line 7
            rep.krylov_mv += 1
            eta1 = C.T @ v                                 # line 7a
            v = v - C @ eta1
            sigma = float(rt @ v)
            if sigma == 0.0:
                status = BREAKDOWN
                break
            alpha = rho / sigma                            # line 8
            s = r - alpha * v
            if _norm(s) == 0.0:                            # lines 9-10a (early exit off [D5]; exact-zero guard)
                x = x + alpha * ph
                xi = xi + alpha * eta1
                r = s
                i += 1
                break
            sh = pc(s)
            t = op.apply(sh)                               # line 12
            rep.krylov_mv += 1
            eta2 = C.T @ t                                 # line 12a
            t = t - C @ eta2
            tau = float(t @ t)
            if tau == 0.0:
                status = BREAKDOWN
                break
            omega = float(t @ s) / tau                     # line 13
            if omega == 0.0:
                status = BREAKDOWN
                break
            xi = xi + alpha * eta1 + omega * eta2          # line 13a
            x = x + alpha * ph + omega * sh                # line 14 [D22]
            r = s - omega * t                              # line 15
            rho_old = rho                                  # line 16
            i += 1
            if hook is not None:
                hook(dict(rho=rho, sigma=sigma, ss=float(s @ s), ts=float(t @ s), tt=tau,
                          rr=float(r @ r), vv=float(v @ v), x=x, xi=xi))
            rep.history.append((rep.krylov_mv, float("nan"), _norm(r)))
            if _norm(r) > prm.divergence * r0n:            # [D17] instability
                status = UNSTABLE
                break
        rep.cycles += i
        rep.xi = xi
        x = x - U @ xi                                     # line 17a
        rtrue = b - op.apply(x)                            # certification [D23]
        rep.op_apps += 1
        rep.final_true_res = _norm(rtrue)
        rep.final_upd_res = _norm(r)
        if status is not None:
            rep.outcome = status
            break
        if rep.final_true_res <= tol * rep.bnorm:
            rep.outcome = CONVERGED
            break
        if rep.krylov_mv >= prm.max_mv:
            rep.outcome = DRIFT if _norm(r) <= tol * rep.bnorm else MAX_MATVECS
            break
        if i == 0:                                         # restart made no progress
            rep.outcome = DRIFT
            break
        # [D23] drift after 17a: restart from x_hat = x
    rep.k_after = U.shape[1]
    return x, U, C, rep


def bicgstab(op, pc, b, prm):
    """Alg. 2 BiCGStab, right preconditioned = rBiCGStab with k = 0."""
    N = b.size
    e = np.zeros((N, 0))
    x, _, _, rep = rbicgstab(op, pc, b, e, e, prm)
    return x, rep


# ------------------------------------------------------- O7 hybrid / sequence
def run_sequence(workload, systems=None, solver=None, callback=None, switchback=False,
                 refresh_on_epoch=False, refresh_every=0):
    """Solve workload.n_systems systems A_e x_t = b_t in order, carrying the
    recycle space.  method 'rgcrot' | 'gmres' | 'bicgstab' | 'hybrid'.
    Hybrid: systems t < n_sw by rGCROT, then rBiCGStab with the
    space frozen; at the switch and at each A epoch C is invalidated and
    rebuilt against the operator of the method in use [D3].

    Hybrid policy options (SPEC hybrid module, reading R16):
      switchback       -- "if convergence is poor ... switch back to rGCROT":
                          an rBiCGStab solve that does not converge (UNSTABLE,
                          BREAKDOWN, MAX_MATVECS, DRIFT) is re-solved from
                          x = 0 by rGCROT, which updates the space; rBiCGStab
                          resumes with the next system.  Both attempts count.
      refresh_on_epoch -- "intermittent solves with rGCROT to update the
                          recycle space ... when the system matrix changes":
                          the first system of every new A epoch after the
                          switch is solved by rGCROT.
      refresh_every    -- n > 0: every n-th system after the switch is solved
                          by rGCROT (SPEC refresh_every_n).
    Returns [(tag, x, report)]; a switched-back system has tag
    'rbicgstab+rgcrot' and a report with the summed counts."""
    from .stencil import Operator
    prm = workload.params
    method = solver or prm.method
    prob = workload.problem()
    T = workload.n_systems if systems is None else systems
    U = C = None
    c_kind = "ahat"            # C spans M^-1 A U (rGCROT) or A U (rBiCGStab) [D3]
    c_epoch = 0
    epoch = -1
    out = []
    op = pc = None
    for t in range(T):
        e = workload.epoch(t)
        new_epoch = e != epoch
        if new_epoch:
            op = Operator.from_problem(prob, epoch=e)
            pc = make_precond(op, prm)
            epoch = e
        if U is None:
            U = np.zeros((op.N, 0))
            C = np.zeros((op.N, 0))
            c_epoch = e
        b = prob.rhs(t).reshape(-1)
        use_rg = method == "rgcrot" or (method == "hybrid" and hybrid_uses_rgcrot(
            t, prm.n_sw, new_epoch and t > 0, refresh_on_epoch, refresh_every))
        if method == "gmres":
            x, rep = gmres(op, pc, b, prm)
            tag = "gmres"
        elif method == "bicgstab":
            x, rep = bicgstab(op, pc, b, prm)
            tag = "bicgstab"
        elif use_rg:
            x, U, C, rep = rgcrot(op, pc, b, U, C, prm, valid=(c_kind == "ahat" and c_epoch == e))
            c_kind, c_epoch = "ahat", e
            tag = "rgcrot"
        else:
            x, U, C, rep = rbicgstab(op, pc, b, U, C, prm, valid=(c_kind == "a" and c_epoch == e))
            c_kind, c_epoch = "a", e
            tag = "rbicgstab"
            if switchback and rep.outcome != CONVERGED:
                x, U, C, rep2 = rgcrot(op, pc, b, U, C, prm, valid=False)
                c_kind = "ahat"
                rep2.krylov_mv += rep.krylov_mv
                rep2.op_apps += rep.op_apps
                rep = rep2
                tag = "rbicgstab+rgcrot"
        out.append((tag, x, rep))
        if callback:
            callback(t, tag, x, U, C, rep)
    return out


def make_precond(op, prm):
    """The preconditioner named by prm.precond: Jacobi(5+1) (optionally block
    Jacobi, R17), multicolour SSOR(5)+1 (R18) or none (identity)."""
    from .stencil import Jacobi, SSOR
    kind = getattr(prm, "precond", "jacobi")
    if kind == "ssor":
        return SSOR(op, prm.sweeps, getattr(prm, "omega_s", 1.0), prm.omega_g)
    if kind == "none":
        return lambda r: np.array(r, dtype=np.float64, copy=True)
    return Jacobi(op, prm.sweeps, prm.omega_l, prm.omega_g, getattr(prm, "zblocks", 1))


def hybrid_uses_rgcrot(t, n_sw, epoch_changed, refresh_on_epoch, refresh_every):
    """Hybrid schedule (R16): rGCROT for t < n_sw, and after the
    switch on the first system of a new A epoch (refresh_on_epoch) or every
    refresh_every-th system; rBiCGStab otherwise."""
    if t < n_sw:
        return True
    if refresh_on_epoch and epoch_changed:
        return True
    return bool(refresh_every) and (t - n_sw) % refresh_every == refresh_every - 1
