"""Pins for oracle O1 (SpMV) and O2 (Jacobi(5+1)) against things other
than the oracle itself: SPEC hand examples, an independent dense
expansion, closed-form eigenpairs, row-sum identities."""
import json
import os

import numpy as np
import pytest

from oracle.stencil import Operator, Jacobi, jacobi, to_dense
from problems import OFFSETS7, OFFSETS19, get_workload
from problems.stencils import PERIODIC_X, PERIODIC_Z, channel19, convection_diffusion_c1, porous7

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "..", "golden", "spec_examples.json")))


def _random_op(nx, ny, nz, periodic, offsets, seed):
    """Random bands honouring boundary truncation."""
    rng = np.random.default_rng(seed)
    S = len(offsets)
    bands = rng.uniform(-1, 1, size=(S, nz, ny, nx))
    bands[0] += 8.0
    k = np.arange(nz)[:, None, None]
    j = np.arange(ny)[None, :, None]
    i = np.arange(nx)[None, None, :]
    for d, (dx, dy, dz) in enumerate(offsets):
        for idx, dd, n, bit in ((i, dx, nx, 1), (j, dy, ny, 2), (k, dz, nz, 4)):
            if dd and not (periodic & bit):
                bad = np.broadcast_to((idx + dd < 0) | (idx + dd >= n), bands[d].shape)
                bands[d][bad] = 0.0
    return Operator(nx, ny, nz, periodic, offsets, bands)


def test_spec_identity_stencil():
    op = Operator(3, 2, 2, 0, OFFSETS7, np.concatenate(
        [np.ones((1, 2, 2, 3)), np.zeros((6, 2, 2, 3))]))
    x = np.arange(12.0) - 4.5
    assert np.array_equal(op.apply(x), x)


def test_spec_poisson1d():
    g = GOLD["matvec_poisson1d_n3"]
    offs = np.array([(0, 0, 0), (-1, 0, 0), (1, 0, 0)], dtype=np.int8)
    b = np.zeros((3, 1, 1, 3))
    b[0] = g["diag"]
    b[1][..., 1:] = g["off"]
    b[2][..., :2] = g["off"]
    op = Operator(3, 1, 1, 0, offs, b)
    assert np.array_equal(op.apply(np.array(g["x"])), np.array(g["y"]))
    g2 = GOLD["dense_poisson1d_n2"]
    b2 = np.zeros((3, 1, 1, 2))
    b2[0] = 2.0
    b2[1][..., 1:] = -1.0
    b2[2][..., :1] = -1.0
    assert np.array_equal(to_dense(Operator(2, 1, 1, 0, offs, b2)), np.array(g2["dense"]))


def test_spec_poisson2d_interior_row():
    g = GOLD["poisson2d_3x3_interior_row"]
    offs = np.array([(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0)], dtype=np.int8)
    b = np.zeros((5, 1, 3, 3))
    b[0] = 4.0
    b[1][..., :, 1:] = -1.0
    b[2][..., :, :2] = -1.0
    b[3][..., 1:, :] = -1.0
    b[4][..., :2, :] = -1.0
    D = to_dense(Operator(3, 3, 1, 0, offs, b))
    row = D[4]
    assert row[4] == g["row_center"]
    assert sorted(row[[1, 3, 5, 7]].tolist()) == g["row_neighbours"]
    assert np.count_nonzero(row) == 5
    assert np.array_equal(D, D.T)                  # S:375 symmetric for Dirichlet


@pytest.mark.parametrize("offsets", [OFFSETS7, OFFSETS19], ids=["7pt", "19pt"])
@pytest.mark.parametrize("periodic", [0, PERIODIC_X, PERIODIC_X | PERIODIC_Z, 7])
def test_spmv_matches_dense_expansion(offsets, periodic):
    op = _random_op(5, 4, 3, periodic, offsets, seed=periodic + len(offsets))
    x = np.random.default_rng(1).uniform(-1, 1, op.N)
    D = to_dense(op)
    np.testing.assert_allclose(op.apply(x), D @ x, rtol=0, atol=1e-13)


def test_spmv_linearity_and_extended_precision():
    op = Operator.from_problem(channel19(8))
    rng = np.random.default_rng(3)
    x, y = rng.uniform(-1, 1, (2, op.N))
    a = 0.37
    lhs = op.apply(a * x + y)
    rhs = a * op.apply(x) + op.apply(y)
    assert np.max(np.abs(lhs - rhs)) <= 1e-13 * np.max(op.apply_abs(np.abs(a * x) + np.abs(y)))
    d = np.abs(op.apply(x) - op.apply_ld(x).astype(np.float64))
    assert np.all(d <= 4e-16 * len(op.offsets) * op.apply_abs(x))


def test_truncation_is_asserted():
    b = np.zeros((7, 2, 2, 2))
    b[0] = 1.0
    b[1] = 1.0                                      # reaches x = -1 at i = 0
    with pytest.raises(AssertionError):
        Operator(2, 2, 2, 0, OFFSETS7, b)


def _c1_eigpair(n, kx, ky, kz, pe=10.0):
    """Closed form: A = sum_d I x T_d x I with T_d tridiagonal Toeplitz
    (sub = -1/h^2 - a_d/h, super = -1/h^2, diag = 2/h^2 + a_d/h).
    Eigenvector  prod_d (sub/super)^(i_d/2) sin(i_d k_d pi h), i_d = 1..n,
    eigenvalue  sum_d [diag_d - 2 sqrt(sub_d super_d) cos(k_d pi h)]."""
    h = 1.0 / (n + 1)
    a = pe * np.array([1.0, 0.5, 0.25])
    lam = 0.0
    vecs = []
    for d, kd in enumerate((kx, ky, kz)):
        sub, sup, dg = -1 / h**2 - a[d] / h, -1 / h**2, 2 / h**2 + a[d] / h
        lam += dg - 2.0 * np.sqrt(sub * sup) * np.cos(kd * np.pi * h)
        i = np.arange(1, n + 1)
        vecs.append((sub / sup) ** (i / 2.0) * np.sin(i * kd * np.pi * h))
    v = vecs[2][:, None, None] * vecs[1][None, :, None] * vecs[0][None, None, :]
    return lam, v.reshape(-1), 6 / h**2 + a.sum() / h


@pytest.mark.parametrize("ks", [(1, 1, 1), (2, 5, 3), (16, 1, 9), (7, 7, 7)])
def test_c1_closed_form_eigenpairs(ks):
    n = 16
    op = Operator.from_problem(convection_diffusion_c1(n))
    lam, v, _ = _c1_eigpair(n, *ks)
    Av = op.apply(v)
    assert np.linalg.norm(Av - lam * v) <= 1e-14 * lam * np.linalg.norm(v) * 10


@pytest.mark.parametrize("ks", [(1, 1, 1), (3, 8, 2), (16, 16, 16)])
def test_jacobi_closed_form_on_c1_eigenvectors(ks):
    """M^-1 v = [1 - (1 - w_g mu)(1 - w_l mu)^5] / lambda v,  mu = lambda/d."""
    n = 16
    op = Operator.from_problem(convection_diffusion_c1(n))
    lam, v, dgl = _c1_eigpair(n, *ks)
    mu = lam / dgl
    c = (1.0 - (1.0 - 1.0 * mu) * (1.0 - 0.8 * mu) ** 5) / lam
    z = jacobi(op, v)
    assert np.linalg.norm(z - c * v) <= 1e-13 * abs(c) * np.linalg.norm(v) * 10


def test_jacobi_diagonal_operator():
    rng = np.random.default_rng(5)
    b = np.zeros((7, 3, 3, 3))
    b[0] = rng.uniform(1, 3, (3, 3, 3))
    op = Operator(3, 3, 3, 0, OFFSETS7, b)
    r = rng.uniform(-1, 1, 27)
    for wl, wg in ((0.8, 1.0), (0.6, 0.5)):
        z = jacobi(op, r, 5, wl, wg)
        np.testing.assert_allclose(z, (1 - (1 - wg) * (1 - wl) ** 5) * r / b[0].reshape(-1),
                                   rtol=1e-15)
    z = jacobi(op, r, 1, 1.0, 1.0)
    np.testing.assert_allclose(z, r / b[0].reshape(-1), rtol=1e-15)


def test_jacobi_unrolled_linear_deterministic():
    """equals an explicitly unrolled 5+1 sweep, is
    linear, and bitwise deterministic.  The unrolled form uses the dense
    matrix, not Operator.apply."""
    op = Operator.from_problem(porous7(12, 2))
    D = to_dense(op)
    dg = np.diag(D)
    rng = np.random.default_rng(11)
    r1, r2 = rng.uniform(-1, 1, (2, op.N))
    z = np.zeros(op.N)
    for s in range(6):
        w = 1.0 if s == 5 else 0.8
        z = z + w * (r1 - D @ z) / dg
    z1 = jacobi(op, r1)
    np.testing.assert_allclose(z1, z, rtol=1e-12, atol=1e-15 * np.abs(z).max())
    np.testing.assert_allclose(jacobi(op, r1 + r2), z1 + jacobi(op, r2), rtol=0,
                               atol=1e-13 * np.abs(z1).max())
    assert np.array_equal(jacobi(op, r1), z1)
    pc = Jacobi(op)
    assert np.array_equal(pc(r1), z1)


def test_channel_operator_row_sums_and_pattern():
    """Laplacian of a constant vanishes: every non-pinned row of the
    channel operator sums to zero (mapped Laplacian kills constants;
    Neumann folding preserves row sums); interior rows have 19 nnz."""
    prob = channel19(12)
    op = Operator.from_problem(prob)
    rs = op.apply(np.ones(op.N))
    scale = np.abs(op.diag()).max()
    rs[0] -= 1.0                                  # pinned identity row
    assert np.max(np.abs(rs)) <= 1e-12 * scale
    nnz = (op.bands != 0).sum(axis=0).reshape(-1)
    j = (np.arange(op.N) // op.nx) % op.ny
    assert np.all(nnz[(j > 0) & (j < op.ny - 1)][1:] == 19)
    D = to_dense(op)
    assert np.linalg.norm(D - D.T) / np.linalg.norm(D) > 1e-3     # nonsymmetric
    assert op.periodic == PERIODIC_X | PERIODIC_Z


def _channel_grid(n, beta=2.0, shear=0.1):
    xi = (np.arange(n) + 0.5) / n
    eta = (np.arange(n) + 0.5) / n
    Y = np.tanh(beta * (2 * eta - 1)) / np.tanh(beta)
    return xi, Y


def test_channel_exact_discrete_fourier_modes():
    """For p = cos(2 pi xi) cos(2 pi zeta) (eta-independent) every
    eta-derivative stencil vanishes exactly (also across the Neumann fold),
    and the xi/zeta stencils give closed forms:
      A p = -(2cos d - 2)/D^2 [(1+a^2) + (1+c^2)] p - 2ac sin x sin z sin^2 d / D^2,
    d = 2 pi D.  Pins the (1+a^2), (1+c^2), 2ac coefficients and the
    periodic wrap."""
    n, a = 16, 0.1
    op = Operator.from_problem(channel19(n))
    Dl = 1.0 / n
    xi = (np.arange(n) + 0.5) / n
    X = 2 * np.pi * xi[None, None, :]
    Z = 2 * np.pi * xi[:, None, None]
    p = (np.cos(X) * np.cos(Z) * np.ones((n, n, n))).reshape(-1)
    d = 2 * np.pi * Dl
    exact = (-(2 * np.cos(d) - 2) / Dl**2 * (2 + 2 * a * a) * np.cos(X) * np.cos(Z)
             - 2 * a * a * np.sin(X) * np.sin(Z) * np.sin(d) ** 2 / Dl**2) * np.ones((n, n, n))
    exact = exact.reshape(-1)
    got = op.apply(p)
    assert np.max(np.abs(got[1:] - exact[1:])) <= 1e-9 * np.max(np.abs(exact))


def test_channel_second_order_consistency():
    """p = cos(2 pi x_phys) with x_phys = xi + a Y(eta) is periodic in xi and
    depends only on the physical x, so -Laplacian p = (2 pi)^2 p.  Away from
    the walls the 19-point operator must reproduce it to O(Delta^2): the
    error ratio between n = 16 and 32 is ~4.  Pins every mapped-coordinate
    term (Y', Y'', the xi-eta cross stencil)."""
    errs = []
    for n in (16, 32):
        op = Operator.from_problem(channel19(n))
        xi, Y = _channel_grid(n)
        xp = xi[None, None, :] + 0.1 * Y[None, :, None]
        p = (np.cos(2 * np.pi * xp) * np.ones((n, 1, 1))).reshape(-1)
        exact = (2 * np.pi) ** 2 * p
        j = (np.arange(op.N) // n) % n
        inner = (j >= n // 4) & (j < n - n // 4)
        inner[0] = False
        errs.append(np.max(np.abs(op.apply(p) - exact)[inner]))
    ratio = errs[0] / errs[1]
    assert 3.0 < ratio < 5.5, (errs, ratio)


def test_porous_operator_properties():
    op = Operator.from_problem(porous7(12, 2))
    D = to_dense(op)
    assert np.all(np.diag(D) > 0)
    # weak diagonal dominance with strict dominance on Dirichlet x rows
    off = np.abs(D).sum(axis=1) - np.abs(np.diag(D))
    assert np.all(np.diag(D) >= off * (1 - 1e-14))
    assert np.linalg.norm(D - D.T) / np.linalg.norm(D) > 1e-2
    # Jacobi iteration matrix contracts (rho(I - 0.8 D^-1 A) < 1)
    J = np.eye(op.N) - 0.8 * D / np.diag(D)[:, None]
    assert np.max(np.abs(np.linalg.eigvals(J))) < 1.0


# ----------------------------------------------------- block Jacobi (R17)
def _block_of(nz, zb, n, nx, ny):
    return (n // (nx * ny)) // zb


@pytest.mark.parametrize("mk,zblocks", [
    (lambda: channel19(8), 2),          # periodic z: the wrap is a block boundary too
    (lambda: porous7(8, 2), 4),
    (lambda: convection_diffusion_c1(8), 2),
])
def test_local_operator_is_block_diagonal_part(mk, zblocks):
    """A_loc (the local sweeps' operator) equals the dense A with every entry
    coupling two different z-blocks removed -- built here from the
    independent per-cell dense expansion and a block-membership mask."""
    from oracle.stencil import local_operator
    prob = mk()
    op = Operator.from_problem(prob)
    A = to_dense(op)
    zb = op.nz // zblocks
    blk = np.arange(op.N) // (op.nx * op.ny) // zb
    mask = blk[:, None] == blk[None, :]
    Aloc = to_dense(local_operator(op, zblocks))
    assert np.array_equal(Aloc, np.where(mask, A, 0.0))
    assert np.count_nonzero(A[~mask]) > 0       # the cut removes something


def test_block_jacobi_matches_dense_sweeps():
    """M^-1 with zblocks = 2 on the channel operator, written out with dense
    matrices: z = w_l D^-1 r, 4x z += w_l D^-1 (r - A_loc z), then
    z += w_g D^-1 (r - A z) (P:146-147 with local sub-domain sweeps)."""
    from oracle.stencil import jacobi
    prob = channel19(8)
    op = Operator.from_problem(prob)
    A = to_dense(op)
    blk = np.arange(op.N) // (op.nx * op.ny) // (op.nz // 2)
    Al = np.where(blk[:, None] == blk[None, :], A, 0.0)
    Dinv = 1.0 / np.diag(A)
    r = np.random.default_rng(7).uniform(-1, 1, op.N)
    z = 0.8 * Dinv * r
    for _ in range(4):
        z = z + 0.8 * Dinv * (r - Al @ z)
    z = z + 1.0 * Dinv * (r - A @ z)
    assert np.allclose(jacobi(op, r, zblocks=2), z, rtol=0, atol=1e-13 * np.abs(z).max())
    assert np.array_equal(jacobi(op, r, zblocks=1), jacobi(op, r))


# ------------------------------------------------------ SSOR (R18)
def test_ssor_diagonal_closed_form():
    """On a diagonal A one forward SOR pass with omega = 1 solves exactly:
    z = D^-1 r, and neither the backward pass nor the global sweep moves it
    (SPEC S:120-style closed form)."""
    from oracle.stencil import ssor
    rng = np.random.default_rng(1)
    nx = ny = nz = 4
    bands = np.zeros((7, nz, ny, nx))
    bands[0] = rng.uniform(1, 3, (nz, ny, nx))
    op = Operator(nx, ny, nz, 0, OFFSETS7, bands)
    r = rng.uniform(-1, 1, op.N)
    assert np.allclose(ssor(op, r, sweeps=1, omega=1.0), r / op.diag(), rtol=0, atol=1e-15)


@pytest.mark.parametrize("mk", [lambda: channel19(8), lambda: porous7(8, 2),
                                lambda: convection_diffusion_c1(8)])
def test_ssor_matches_block_triangular_formula(mk):
    """Multicolour SSOR written as matrices: with the colour order of
    colour_of, L / U = the couplings to earlier / later colours of the dense
    expansion, one symmetric sweep is z <- z + (D/w + L)^-1 (r - A z), then
    z <- z + (D/w + U)^-1 (r - A z) (triangular solves, an independent code
    path from the colour loop), and the global sweep z += w_g D^-1 (r - A z)."""
    import scipy.linalg as sla
    from oracle.stencil import colour_of, ssor
    prob = mk()
    op = Operator.from_problem(prob)
    A = to_dense(op)
    col = colour_of(op)
    perm = np.argsort(col, kind="stable")
    Ap = A[np.ix_(perm, perm)]
    cp = col[perm]
    D = np.diag(np.diag(Ap))
    L = np.where(cp[:, None] > cp[None, :], Ap, 0.0)
    U = np.where(cp[:, None] < cp[None, :], Ap, 0.0)
    assert np.count_nonzero(np.where(cp[:, None] == cp[None, :], Ap, 0.0) - D) == 0   # colours decouple
    w = 1.1
    r = np.random.default_rng(3).uniform(-1, 1, op.N)
    rp = r[perm]
    z = np.zeros(op.N)
    for _ in range(3):
        z = z + sla.solve_triangular(D / w + L, rp - Ap @ z, lower=True)
        z = z + sla.solve_triangular(D / w + U, rp - Ap @ z, lower=False)
    z = z + (rp - Ap @ z) / np.diag(Ap)
    out = np.empty(op.N)
    out[perm] = z
    ref = ssor(op, r, sweeps=3, omega=w)
    assert np.allclose(ref, out, rtol=0, atol=1e-12 * np.abs(out).max())


@pytest.mark.parametrize("mk", [lambda: channel19(8), lambda: porous7(10, 2),
                                lambda: convection_diffusion_c1(6)])
def test_to_sparse_equals_dense_expansion(mk):
    """oracle.stencil.to_sparse (the sparse-LU reference of reading R12) is
    the per-cell dense expansion to_dense, entry for entry."""
    from oracle.stencil import to_sparse
    op = Operator.from_problem(mk())
    assert np.array_equal(to_sparse(op).toarray(), to_dense(op))
