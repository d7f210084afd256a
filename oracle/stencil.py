"""Oracle O1 (stencil SpMV) and O2 (Jacobi(5+1) preconditioner).  TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

O1  y_n = sum_d a_d[n] * x[nbr(n, d)]                      (
    PAPER P:121-123 banded storage).  nbr wraps on periodic axes; on a
    non-periodic axis an out-of-grid neighbour must carry a zero
    coefficient -- asserted at construction.
O2  "Five sweeps of the Jacobi method with a relaxation parameter ...
    followed by a sweep of point Jacobi smoothing on the global domain"
    (P:147), from z = 0:
        z = w_l D^-1 r;  4x: z += w_l D^-1 (r - A z);  1x: z += w_g D^-1 (r - A z)
    w_l = 0.8, w_g = 1.0, all sweeps global (reading R3).

Pins (tests/oracle/test_stencil_pins.py): dense expansion built by
explicit per-cell loops; SPEC's hand examples;
the closed-form eigenpairs of the c1 operator (Kronecker sum of
tridiagonal Toeplitz matrices); zero row sums of the channel operator;
Jacobi on a diagonal A and on the c1 eigenvectors (closed form
[1 - (1-w_g mu)(1-w_l mu)^5]/lambda).
"""
import numpy as np


def shifted(x3, dx, dy, dz, periodic):
    """xs[k, j, i] = x3[k+dz, j+dy, i+dx]; wraps on periodic axes, 0 outside."""
    out = x3
    for axis, d, bit in ((2, dx, 1), (1, dy, 2), (0, dz, 4)):
        if d == 0:
            continue
        if periodic & bit:
            out = np.roll(out, -d, axis=axis)
        else:
            n = out.shape[axis]
            res = np.zeros_like(out)
            src = [slice(None)] * 3
            dst = [slice(None)] * 3
            if d > 0:
                src[axis] = slice(d, n)
                dst[axis] = slice(0, n - d)
            else:
                src[axis] = slice(0, n + d)
                dst[axis] = slice(-d, n)
            res[tuple(dst)] = out[tuple(src)]
            out = res
    return out


class Operator:
    """Banded structured-grid operator A (bands [S, nz, ny, nx], x-fastest)."""

    def __init__(self, nx, ny, nz, periodic, offsets, bands, check=True):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.periodic = int(periodic)
        self.offsets = np.asarray(offsets, dtype=np.int64)
        self.bands = np.asarray(bands, dtype=np.float64).reshape(
            len(self.offsets), self.nz, self.ny, self.nx)
        self.N = self.nx * self.ny * self.nz
        d0 = [d for d, o in enumerate(self.offsets) if tuple(o) == (0, 0, 0)]
        assert len(d0) == 1, "exactly one diagonal band (S:38)"
        self.d0 = d0[0]
        if check:
            self._check_truncation()

    @classmethod
    def from_problem(cls, prob, epoch=0):
        return cls(prob.nx, prob.ny, prob.nz, prob.periodic, prob.offsets,
                   prob.bands(epoch=epoch))

    def _check_truncation(self):
        k = np.arange(self.nz)[:, None, None]
        j = np.arange(self.ny)[None, :, None]
        i = np.arange(self.nx)[None, None, :]
        for d, (dx, dy, dz) in enumerate(self.offsets):
            bad = np.zeros((self.nz, self.ny, self.nx), dtype=bool)
            for idx, dd, n, bit in ((i, dx, self.nx, 1), (j, dy, self.ny, 2), (k, dz, self.nz, 4)):
                if dd and not (self.periodic & bit):
                    bad |= np.broadcast_to((idx + dd < 0) | (idx + dd >= n), bad.shape)
            assert not np.any(self.bands[d][bad]), \
                f"band {d} reaches outside a non-periodic axis (S:39)"

    def diag(self):
        return self.bands[self.d0].reshape(-1)

    def apply(self, x):
        """O1: y = A x."""
        x3 = np.asarray(x, dtype=np.float64).reshape(self.nz, self.ny, self.nx)
        y = np.zeros_like(x3)
        for d, (dx, dy, dz) in enumerate(self.offsets):
            y += self.bands[d] * shifted(x3, dx, dy, dz, self.periodic)
        return y.reshape(-1)

    def apply_ld(self, x):
        """O1 in extended precision (np.longdouble accumulation) -- the
        per-kernel reference for the 1e-12 componentwise check."""
        x3 = np.asarray(x, dtype=np.longdouble).reshape(self.nz, self.ny, self.nx)
        y = np.zeros_like(x3)
        for d, (dx, dy, dz) in enumerate(self.offsets):
            y += self.bands[d].astype(np.longdouble) * shifted(x3, dx, dy, dz, self.periodic)
        return y.reshape(-1)

    def apply_abs(self, x):
        """(|A| |x|)_n, the scale of the componentwise SpMV tolerance (D25)."""
        x3 = np.abs(np.asarray(x, dtype=np.float64)).reshape(self.nz, self.ny, self.nx)
        y = np.zeros_like(x3)
        for d, (dx, dy, dz) in enumerate(self.offsets):
            y += np.abs(self.bands[d]) * shifted(x3, dx, dy, dz, self.periodic)
        return y.reshape(-1)


def to_dense(op, cap=8192):
    """Dense N x N expansion built cell by cell; an
    independent construction used to pin Operator.apply."""
    N = op.N
    assert N <= cap, "dense expansion only for tiny grids"
    Ad = np.zeros((N, N))
    for k in range(op.nz):
        for j in range(op.ny):
            for i in range(op.nx):
                n = i + op.nx * (j + op.ny * k)
                for d, (dx, dy, dz) in enumerate(op.offsets):
                    ii, jj, kk = i + dx, j + dy, k + dz
                    ok = True
                    for v, nn, bit in ((ii, op.nx, 1), (jj, op.ny, 2), (kk, op.nz, 4)):
                        if not (0 <= v < nn) and not (op.periodic & bit):
                            ok = False
                    if not ok:
                        continue
                    ii %= op.nx
                    jj %= op.ny
                    kk %= op.nz
                    Ad[n, ii + op.nx * (jj + op.ny * kk)] += op.bands[d, k, j, i]
    return Ad


def to_sparse(op):
    """A as a scipy CSR matrix, assembled band by band with to_dense's
    per-cell rule (wrap on periodic axes, drop out-of-grid neighbours),
    vectorised: the direct-solve reference for grids too large for
    to_dense (sparse LU up to 32^3)."""
    import scipy.sparse as sp
    k, j, i = np.meshgrid(np.arange(op.nz), np.arange(op.ny), np.arange(op.nx), indexing="ij")
    rows, cols, vals = [], [], []
    n = (i + op.nx * (j + op.ny * k)).ravel()
    for d, (dx, dy, dz) in enumerate(op.offsets):
        ii, jj, kk = i + dx, j + dy, k + dz
        ok = np.ones(ii.shape, dtype=bool)
        for v, nn, bit in ((ii, op.nx, 1), (jj, op.ny, 2), (kk, op.nz, 4)):
            if not (op.periodic & bit):
                ok &= (v >= 0) & (v < nn)
        m = ok.ravel()
        col = ((ii % op.nx) + op.nx * ((jj % op.ny) + op.ny * (kk % op.nz))).ravel()
        rows.append(n[m])
        cols.append(col[m])
        vals.append(op.bands[d].ravel()[m])
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(op.N, op.N))


def local_operator(op, zblocks):
    """A_loc: A with every coupling between different z-blocks removed.  The
    z axis is cut into `zblocks` equal slabs (planes [b nz/P, (b+1) nz/P),
    the rank decomposition of SURVEY §8(e)); a band reaching across a slab
    boundary (including the periodic wrap) gets a zero coefficient there, so
    A_loc is block diagonal with the diagonal blocks of A (overlapping
    Schwarz with zero overlap)."""
    assert op.nz % zblocks == 0, "z-blocks must divide nz"
    zb = op.nz // zblocks
    bands = op.bands.copy()
    k = np.arange(op.nz)
    for d, (dx, dy, dz) in enumerate(op.offsets):
        if dz == 0:
            continue
        cross = ((k + dz) // zb != k // zb) | (k + dz < 0) | (k + dz >= op.nz)
        bands[d][cross] = 0.0
    per = op.periodic & ~4 if zblocks > 1 else op.periodic
    return Operator(op.nx, op.ny, op.nz, per, op.offsets, bands)


def jacobi(op, r, sweeps=5, omega_l=0.8, omega_g=1.0, zblocks=1):
    """O2: z ~= M^-1 r by `sweeps` under-relaxed Jacobi sweeps from z = 0
    followed by one point-Jacobi sweep with omega_g.  With
    zblocks > 1 the `sweeps` relaxed sweeps are the paper's "sweeps on the
    local sub-domains" -- they use A_loc (local_operator: no coupling between
    z-blocks, so no communication between ranks owning whole blocks) -- and
    the last sweep is the global one (reading R17)."""
    D = op.diag()
    r = np.asarray(r, dtype=np.float64)
    A_l = op if zblocks <= 1 else local_operator(op, zblocks)
    z = omega_l * r / D                              # first sweep from z = 0
    for _ in range(sweeps - 1):
        z = z + omega_l * (r - A_l.apply(z)) / D
    z = z + omega_g * (r - op.apply(z)) / D          # global point-Jacobi sweep
    return z


def colour_of(op):
    """Multicolour ordering for the SSOR sweeps (reading R18): colour =
    (i mod 2) + 2 (j mod 2) + 4 (k mod 2).  Any two cells coupled by a
    stencil offset in {-1,0,1}^3 differ by one in some coordinate, so their
    colours differ: a colour's cells can be updated together."""
    k, j, i = np.meshgrid(np.arange(op.nz), np.arange(op.ny), np.arange(op.nx), indexing="ij")
    return ((i & 1) + 2 * (j & 1) + 4 * (k & 1)).reshape(-1)


def ssor(op, r, sweeps=5, omega=1.0, omega_g=1.0):
    """SSOR smoothing preconditioner ("5 inner iterations of ...
    SSOR smoothing"; "one forward SOR sweep then one backward SOR
    sweep per sweep count"), from z = 0, in the multicolour order of
    colour_of (forward: colours 0..7, backward: 7..0; Gauss-Seidel within
    the ordering = cells of one colour at a time), followed by the global
    point-Jacobi sweep of the Jacobi variant.  Reading R18."""
    D = op.diag()
    r = np.asarray(r, dtype=np.float64)
    col = colour_of(op)
    masks = [col == c for c in range(8)]
    z = np.zeros_like(r)
    for _ in range(sweeps):
        for order in (range(8), range(7, -1, -1)):
            for c in order:
                m = masks[c]
                if not m.any():
                    continue
                res = r - op.apply(z)
                z[m] = z[m] + omega * res[m] / D[m]
    z = z + omega_g * (r - op.apply(z)) / D
    return z


class SSOR:
    """The SSOR(sweeps)+1 preconditioner as a callable (a fixed linear map)."""

    def __init__(self, op, sweeps=5, omega=1.0, omega_g=1.0):
        self.op, self.sweeps, self.omega, self.omega_g = op, sweeps, omega, omega_g

    def __call__(self, r):
        return ssor(self.op, r, self.sweeps, self.omega, self.omega_g)


class Jacobi:
    """The preconditioner as a callable r -> M^-1 r (a fixed linear map)."""

    def __init__(self, op, sweeps=5, omega_l=0.8, omega_g=1.0, zblocks=1):
        self.op, self.sweeps, self.omega_l, self.omega_g = op, sweeps, omega_l, omega_g
        self.zblocks = zblocks

    def __call__(self, r):
        return jacobi(self.op, r, self.sweeps, self.omega_l, self.omega_g, self.zblocks)
