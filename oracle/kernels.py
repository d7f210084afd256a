"""Oracle per-kernel references: the operations the solvers' block and
rBiCGStab kernels perform, each written out as its plain definition.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Each function is one step of PAPER.md Alg. 3 / Alg. 4 taken on its own
(the rGCROT / rBiCGStab iterations of oracle/krylov.py perform the same
steps inline).  Inner products accumulate in np.longdouble (SURVEY §8(c)
"per-kernel references accumulate in np.longdouble"); everything else is
fp64 in the order the definition states.  Vectors are 1-D float64 arrays,
Q a list of them (the columns of [C V_j], U or C).

Pins (tests/oracle/test_kernel_pins.py):
  * block_dot: exact rational arithmetic (fractions.Fraction) on small
    inputs, rounded once;
  * block_project: with an orthonormal Q the result is orthogonal to every
    column and w = w_new + Q eta (the projector identity of eq. (8));
  * gram_update: with G the exact Gram matrix of Q, h = 2 g - G g equals
    the coefficients of two classical Gram-Schmidt passes, g1 + Q^T (w - Q
    g1) (the algebra DESIGN.md R19 rests on), computed independently here
    in exact rational arithmetic; with G = I it is block_update(Q, g, w);
  * normalize: unit norm, and the D18 breakdown branch;
  * project_update, lincomb, rotate: exact rational arithmetic;
  * bicg_p, bicg_project_s, bicg_xr (with block_dot / block_update for
    line 12a) composed into whole iterations reproduce oracle.krylov.
    rbicgstab's per-iteration scalars and iterates, whose iterates are in
    turn pinned to scipy's BiCGStab (test_krylov_pins).
"""
import numpy as np

LD = np.longdouble


def _dot(a, b):
    return float(np.dot(np.asarray(a, dtype=LD), np.asarray(b, dtype=LD)))


# ------------------------------------------------ Alg. 3 lines 6a-9, Alg. 4 7a / 12a
def block_dot(Q, w):
    """[C V_j]^T w (Alg. 3 line 6a B(:,j) = C^T w and lines 7-8 h_ij =
    v_i^T w; Alg. 4 lines 7a / 12a eta = C^T v)."""
    return np.array([_dot(q, w) for q in Q])


def block_update(Q, g, w, dots=()):
    """w - sum_c g_c Q_c (Alg. 3 lines 6c / 9, Alg. 4 lines 7a / 12a), then
    the inner products of the new w with each vector of `dots` (None = w)."""
    wn = w.copy()
    for c, q in enumerate(Q):
        wn = wn - g[c] * q
    return wn, [(_dot(wn, wn) if d is None else _dot(wn, d)) for d in dots]


def block_project(Q, w):
    """eta = Q^T w; w <- w - Q eta (the recycle projection of Alg. 3 lines
    1b / 6a-6c and Alg. 4 lines 1c / 7a / 12a, i.e. (I - C C^T) w, eq. (8));
    returns (eta, w_new, ||w_new||^2)."""
    eta = block_dot(Q, w)
    wn, (nn,) = block_update(Q, eta, w, (None,))
    return eta, wn, nn


def gram_matrix(ncol, k, grow):
    """The Gram matrix the Gram-corrected update uses (R19):
    the leading k x k block (C^T C) is I; rows i >= k hold the lagged inner
    products grow[i][l] = q_i^T q_l for l <= i, mirrored."""
    G = np.zeros((ncol, ncol))
    for i in range(ncol):
        for l in range(ncol):
            if i < k and l < k:
                G[i, l] = 1.0 if i == l else 0.0
            elif i >= l:
                G[i, l] = grow[i][l]
            else:
                G[i, l] = grow[l][i]
    return G


def gram_update(Q, k, g, grow, w):
    """DESIGN.md R19: h = 2 g - G g with G = gram_matrix(k, grow) (the two
    classical Gram-Schmidt passes' coefficients g1 + Q^T(w - Q g1) written
    with the Gram matrix, g1 = g = Q^T w); w <- w - Q h.  Returns (h, w_new,
    ||w_new||^2)."""
    G = gram_matrix(len(Q), k, grow)
    h = np.array([2.0 * g[c] - _dot(G[c], g) for c in range(len(Q))])
    wn, (nn,) = block_update(Q, h, w, (None,))
    return h, wn, nn


def project_update(C, U, xi, r, x=None):
    """Alg. 3 line 1b / Alg. 4 line 1c (reading D20: also at every cycle
    start): r <- r - C xi, x <- x + U xi.  Returns (r_new, x_new or None,
    ||r_new||^2)."""
    rn = r.copy()
    for c, q in enumerate(C):
        rn = rn - xi[c] * q
    xn = None
    if x is not None:
        xn = x.copy()
        for c, u in enumerate(U):
            xn = xn + xi[c] * u
    return rn, xn, _dot(rn, rn)


def normalize(w, nrm2, nin2=None):
    """Alg. 3 line 10: v_{j+1} = w / h_{j+1,j}, h = sqrt(nrm2); happy
    breakdown (reading D18) when h <= 1e-14 sqrt(nin2): v = 0, flag 1."""
    h = np.sqrt(nrm2)
    if nin2 is not None and not (h > 1e-14 * np.sqrt(nin2)):
        return np.zeros_like(w), 1.0
    return w / h, 0.0


def lincomb(Q, coef, outs, scale, acc):
    """out_o = scale_o * sum_c coef[o][c] Q_c (+ out_o when acc_o): the
    cycle-end update x += V_m y - U (B y) (Alg. 3 lines 13-13a, eq. (6)) and
    the line-14a extension vectors."""
    res = []
    for o in range(len(outs)):
        s = np.zeros_like(Q[0])
        for c, q in enumerate(Q):
            s = s + coef[o][c] * q
        v = scale[o] * s
        res.append(outs[o] + v if acc[o] else v)
    return res


def rotate(Q, T, kout=None):
    """[q_0 .. q_{k-1}] T, first kout columns (line 1a U <- U R^-1, C <- C~
    R^-1; the line-14a truncation).  T is k x k (T[l][c] multiplies q_l
    into column c)."""
    k = len(Q)
    kout = k if kout is None else kout
    return [sum(T[l][c] * Q[l] for l in range(k)) for c in range(kout)]


# ------------------------------------------------------------ Alg. 4 (rBiCGStab)
def bicg_p(first, r, p, v, invD, omega_l, cur, prev, thr_conv, thr_div):
    """Alg. 4 line 6 and the first Jacobi sweep of p_hat = M^-1 p (right
    preconditioning, D2): p = r (i = 0) or p = r + beta (p - omega v) with
    beta = (rho_i / rho_{i-1}) (alpha_{i-1} / omega_{i-1}); z = w_l p / D
    (invD = 1/D, or None: z = p).  The stop test of the lookahead (DESIGN
    §7): line 3 (||r|| > tol ||b||), line 5 (rho == 0), the previous
    iteration's breakdown / exit flags and the D17 divergence bound.
    Returns (stop, p, z)."""
    if not first:
        rn = np.sqrt(cur["rr"])
        stop = (prev["flag"] != 0.0 or prev["sigma"] == 0.0 or not (rn > thr_conv)
                or cur["rho"] == 0.0 or not (rn <= thr_div))
        if stop:
            return True, p, None
        alpha = prev["rho"] / prev["sigma"]
        omega = prev["ts"] / prev["tt"]
        beta = (cur["rho"] / prev["rho"]) * (alpha / omega)
        pn = r + beta * (p - omega * v)
    else:
        pn = r.copy()
    z = pn.copy() if invD is None else (omega_l * pn) * invD
    return False, pn, z


def bicg_s(r, v, invD, omega_l, rho, sigma):
    """Alg. 4 line 8 and the first sweep of s_hat: alpha = rho / sigma,
    s = r - alpha v, z = w_l s / D; returns (s, z, ||s||^2)."""
    alpha = rho / sigma
    s = r - alpha * v
    z = s.copy() if invD is None else (omega_l * s) * invD
    return s, z, _dot(s, s)


def bicg_project_s(C, v, rt, r, invD, omega_l, rho):
    """Alg. 4 lines 7a + 8 (R20): eta = C^T v, v <- v - C eta,
    sigma = r~^T v (of the projected v), then line 8.  Returns (eta, v_new,
    sigma, s, z, ||s||^2)."""
    eta, vn, _ = block_project(C, v)
    sigma = _dot(rt, vn)
    s, z, ss = bicg_s(r, vn, invD, omega_l, rho, sigma)
    return eta, vn, sigma, s, z, ss


def bicg_xr(x, r, s, t, ph, sh, rt, cur, xi=None, eta1=None, eta2=None):
    """Alg. 4 lines 13-15 (+ 10-10a exact exit) with the breakdown guards
    of reading D17: alpha = rho/sigma, omega = t^T s / t^T t; mode 2 (no
    update) when sigma = 0, or t^T t = 0 / omega = 0 with s != 0; mode 1
    (exact exit, ||s|| = 0): x += alpha p_hat, r = s; mode 0: x += alpha
    p_hat + omega s_hat, r = s - omega t; line 13a xi += alpha eta1 +
    omega eta2.  Returns (mode, x, r, xi, r~^T r, ||r||^2)."""
    sigma, ss, ts, tt = cur["sigma"], cur["ss"], cur["ts"], cur["tt"]
    if sigma == 0.0:
        mode = 2
    else:
        alpha = cur["rho"] / sigma
        omega = ts / tt if tt != 0.0 else 0.0
        if ss == 0.0:
            mode = 1
        elif tt == 0.0 or omega == 0.0:
            mode = 2
        else:
            mode = 0
    xn, rn = x.copy(), r.copy()
    xin = None if xi is None else xi.copy()
    if mode == 0:
        xn = x + alpha * ph + omega * sh
        rn = s - omega * t
        if xi is not None:
            xin = xi + alpha * eta1 + omega * eta2
    elif mode == 1:
        xn = x + alpha * ph
        rn = s.copy()
        if xi is not None:
            xin = xi + alpha * eta1
    return mode, xn, rn, xin, _dot(rt, rn), _dot(rn, rn)
