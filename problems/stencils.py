"""Banded stencil operators on structured grids (the system matrices A).

Storage ("structured banded sparse storage format ...
only the coefficients for the 7 or 19 point stencil"; SPEC.md S:35-41,
S:82): S separate band arrays of N coefficients (struct of arrays), cell
order x-fastest, n = i + nx*(j + ny*k).  Band d multiplies the neighbour
at offset offsets[d] = (dx, dy, dz); a coefficient that would reach
outside a non-periodic axis is exactly 0.

Three synthetic families stand in for the paper's GenIDLEST systems
(each reading flagged in DESIGN.md "Input recipe"):

* convection_diffusion_c1 -- BASELINE configs[0]: -Laplacian + first-order
  upwind convection, Dirichlet, vertex-centred, h = 1/(n+1).
* channel19 -- configs[1]/[3]: 19-point -Laplacian in a sheared,
  tanh-stretched mapping (P:122-123 ties 19 points to non-orthogonal grids),
  periodic x/z, Neumann y walls, one pinned dof.
* porous7 -- configs[2]/[4]: 7-point variable-coefficient diffusion
  (kappa = 1e-4 in overlapping solid spheres, harmonic-mean faces) plus
  upwind convection, Dirichlet x faces, Neumann y/z faces.
"""
import math
from dataclasses import dataclass, field

import numpy as np

from .rng import uniform, uniform01

# (dx, dy, dz) for each band; band 0 is the diagonal.
OFFSETS7 = np.array(
    [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)],
    dtype=np.int8,
)
OFFSETS19 = np.array(
    [(0, 0, 0),
     (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1),
     (-1, -1, 0), (1, -1, 0), (-1, 1, 0), (1, 1, 0),      # xy edges
     (0, -1, -1), (0, 1, -1), (0, -1, 1), (0, 1, 1),      # yz edges
     (-1, 0, -1), (1, 0, -1), (-1, 0, 1), (1, 0, 1)],     # xz edges
    dtype=np.int8,
)

PERIODIC_X, PERIODIC_Y, PERIODIC_Z = 1, 2, 4


@dataclass
class StencilProblem:
    """A structured-grid operator plus its right-hand-side recipe.

    bands(z0, z1, epoch) returns float64 [S, z1-z0, ny, nx] for the global
    planes [z0, z1) -- a rank generates only its own slab, identical to the
    corresponding planes of the single-GPU array.
    """
    name: str
    nx: int
    ny: int
    nz: int
    periodic: int
    offsets: np.ndarray
    _band_fn: object = field(repr=False)
    rhs_kind: str = "plain"          # "single" | "sequence" | "sequence_meanfree"
    pinned: int = -1                  # global index of the pinned dof, or -1
    info: dict = field(default_factory=dict)

    @property
    def N(self):
        return self.nx * self.ny * self.nz

    @property
    def S(self):
        return len(self.offsets)

    def bands(self, z0=0, z1=None, epoch=0):
        z1 = self.nz if z1 is None else z1
        a = self._band_fn(z0, z1)
        if epoch > 0:
            # A-epoch perturbation: every non-pinned
            # coefficient times (1 + 1e-3 u(3000+e, n*S + d)).
            S = self.S
            P = self.nx * self.ny
            n = np.arange(z0 * P, z1 * P, dtype=np.uint64)
            for d in range(S):
                f = 1.0 + 1e-3 * uniform(3000 + epoch, n * np.uint64(S) + np.uint64(d))
                a[d] *= f.reshape(z1 - z0, self.ny, self.nx)
            self._apply_pin(a, z0, z1)
        return a

    def _apply_pin(self, a, z0, z1):
        if self.pinned < 0:
            return
        P = self.nx * self.ny
        kz = self.pinned // P
        if z0 <= kz < z1:
            rem = self.pinned - kz * P
            j, i = divmod(rem, self.nx)
            a[:, kz - z0, j, i] = 0.0
            a[0, kz - z0, j, i] = 1.0

    def rhs(self, t, z0=0, z1=None):
        """b_t for global planes [z0, z1) (x0 = 0, r0 = b)."""
        z1 = self.nz if z1 is None else z1
        P = self.nx * self.ny
        n = np.arange(z0 * P, z1 * P, dtype=np.uint64)
        b = uniform(0, n)
        if self.rhs_kind != "single":
            # b_t = b0 + 0.05 t noise_t, fresh noise per t
            b = b + (0.05 * t) * uniform(1000 + t, n)
        if self.rhs_kind == "sequence_meanfree":
            mean = self._global_mean(t)
            b = b - mean
            if self.pinned >= 0 and z0 * P <= self.pinned < z1 * P:
                b[self.pinned - z0 * P] = 0.0
        return b.reshape(z1 - z0, self.ny, self.nx)

    def _global_mean(self, t):
        """Mean of b0 + 0.05 t noise_t over the non-pinned cells, computed
        in a fixed plane-chunk order so every rank gets the same bits."""
        P = self.nx * self.ny
        chunk = max(1, (1 << 22) // P)
        acc = 0.0
        for za in range(0, self.nz, chunk):
            zb = min(self.nz, za + chunk)
            n = np.arange(za * P, zb * P, dtype=np.uint64)
            v = uniform(0, n) + (0.05 * t) * uniform(1000 + t, n)
            if self.pinned >= 0 and za * P <= self.pinned < zb * P:
                v[self.pinned - za * P] = 0.0
            acc += float(np.sum(v))
        cnt = self.N - (1 if self.pinned >= 0 else 0)
        return acc / cnt


# ---------------------------------------------------------------- c1 family
def convection_diffusion_c1(n=16, pe=10.0, nx=None, ny=None, nz=None):
    """BASELINE configs[0]: vertex-centred interior nodes 1..n, h = 1/(n+1),
    Dirichlet 0; A = -Lap_h + first-order upwind a.grad, a = Pe (1, .5, .25):
    diag 6/h^2 + sum(a)/h, backward neighbour -1/h^2 - a_d/h, forward -1/h^2."""
    nx = nx or n
    ny = ny or n
    nz = nz or n
    h = 1.0 / (n + 1)
    a = pe * np.array([1.0, 0.5, 0.25])

    def fn(z0, z1):
        nzc = z1 - z0
        out = np.zeros((7, nzc, ny, nx))
        out[0] = 6.0 / h**2 + a.sum() / h
        k = np.arange(z0, z1)[:, None, None]
        j = np.arange(ny)[None, :, None]
        i = np.arange(nx)[None, None, :]
        shape = (nzc, ny, nx)
        for d, (idx, nd) in enumerate(((i, nx), (j, ny), (k, nz))):
            back = np.broadcast_to(idx > 0, shape)
            fwd = np.broadcast_to(idx < nd - 1, shape)
            out[1 + 2 * d] = np.where(back, -1.0 / h**2 - a[d] / h, 0.0)
            out[2 + 2 * d] = np.where(fwd, -1.0 / h**2, 0.0)
        return out

    return StencilProblem(
        name=f"convdiff{nx}x{ny}x{nz}", nx=nx, ny=ny, nz=nz, periodic=0,
        offsets=OFFSETS7.copy(), _band_fn=fn, rhs_kind="single",
        info={"h": h, "a": a.tolist(), "pe": pe},
    )


# ------------------------------------------------------------ channel family
def channel19(n=64, beta=2.0, shear=0.1):
    """BASELINE configs[1]/[3]: cell-centred n^3, Delta = 1/n, eta_j = (j+1/2)/n.
    Mapping x = xi + a Y, y = Y(eta) = tanh(beta(2 eta - 1))/tanh(beta),
    z = zeta + c Y with a = c = shear.  A = -(Laplacian in mapped coords):
      (1+a^2) p_xixi + p_etaeta / Y'^2 - (Y''/Y'^3) p_eta + (1+c^2) p_zz
      - (2a/Y') p_xieta - (2c/Y') p_zeta eta + 2ac p_xizeta
    central differences (4-point cross stencils).  Periodic xi, zeta;
    Neumann eta by mirror ghost (j = -1 / n folded onto j = 0 / n-1);
    cell 0 pinned (identity row, b[0] = 0)."""
    nx = ny = nz = n
    D = 1.0 / n
    aa = cc = shear
    eta = (np.arange(ny) + 0.5) / n
    arg = beta * (2.0 * eta - 1.0)
    th = math.tanh(beta)
    sech2 = 1.0 / np.cosh(arg) ** 2
    Yp = 2.0 * beta * sech2 / th
    Ypp = -8.0 * beta**2 * sech2 * np.tanh(arg) / th

    # coefficients of the Laplacian L, per j (then A = -L)
    L = np.zeros((19, ny))
    inv = 1.0 / D**2
    L[0] = -2.0 * (1 + aa**2) * inv - 2.0 / (Yp**2) * inv - 2.0 * (1 + cc**2) * inv
    L[1] = L[2] = (1 + aa**2) * inv
    L[5] = L[6] = (1 + cc**2) * inv
    L[3] = 1.0 / (Yp**2) * inv + Ypp / (Yp**3) / (2.0 * D)   # -y
    L[4] = 1.0 / (Yp**2) * inv - Ypp / (Yp**3) / (2.0 * D)   # +y
    kxy = -(2.0 * aa / Yp) / (4.0 * D**2)
    kzy = -(2.0 * cc / Yp) / (4.0 * D**2)
    kxz = 2.0 * aa * cc / (4.0 * D**2)
    for d in range(7, 19):
        dx, dy, dz = (int(v) for v in OFFSETS19[d])
        if dz == 0:
            L[d] = kxy * dx * dy
        elif dx == 0:
            L[d] = kzy * dz * dy
        else:
            L[d] = np.full(ny, kxz * dx * dz)
    A = -L
    # Neumann fold: at j = 0 move every dy = -1 coefficient onto dy = 0 (same dx,dz);
    # at j = ny-1 move dy = +1 onto dy = 0.
    idx = {tuple(int(v) for v in o): d for d, o in enumerate(OFFSETS19)}
    for d, o in enumerate(OFFSETS19):
        dx, dy, dz = (int(v) for v in o)
        if dy == -1:
            t = idx[(dx, 0, dz)]
            A[t, 0] += A[d, 0]
            A[d, 0] = 0.0
        if dy == 1:
            t = idx[(dx, 0, dz)]
            A[t, ny - 1] += A[d, ny - 1]
            A[d, ny - 1] = 0.0

    prob = None

    def fn(z0, z1):
        out = np.empty((19, z1 - z0, ny, nx))
        out[:] = A[:, None, :, None]
        prob._apply_pin(out, z0, z1)
        return out

    prob = StencilProblem(
        name=f"channel{n}", nx=nx, ny=ny, nz=nz,
        periodic=PERIODIC_X | PERIODIC_Z, offsets=OFFSETS19.copy(), _band_fn=fn,
        rhs_kind="sequence_meanfree", pinned=0,
        info={"beta": beta, "shear": shear},
    )
    return prob


# ------------------------------------------------------------- porous family
def sphere_centres(n, radius, seed=1, void=0.25):
    """Boolean overlapping spheres with centres uniform in
    [-r, n+r)^3, drawn from seed 1 as a stream of (x, y, z) triples.  For a
    Boolean (Poisson) sphere model the expected void fraction is
    exp(-count V / L^3) with L = n + 2r the side of the box the centres are
    drawn from, so count = ceil(-ln(void) (n+2r)^3 / (4/3 pi r^3)) gives the
    25 % void of BASELINE configs[2] (reading R7; SURVEY's n^3
    count would give ~35 % void).  The achieved fraction is reported."""
    L = n + 2 * radius
    count = int(math.ceil(-math.log(void) * L**3 / (4.0 / 3.0 * math.pi * radius**3)))
    u = uniform01(seed, np.arange(3 * count, dtype=np.uint64)).reshape(count, 3)
    return -radius + (n + 2 * radius) * u


def solid_mask(n, radius, centres, z0, z1):
    """solid[k - z0, j, i] = any sphere with |(i,j,k) - c|^2 < r^2."""
    m = np.zeros((z1 - z0, n, n), dtype=bool)
    r2 = float(radius) ** 2
    for cx, cy, cz in centres:
        ka, kb = max(z0, int(math.floor(cz - radius))), min(z1, int(math.ceil(cz + radius)) + 1)
        if ka >= kb:
            continue
        ja, jb = max(0, int(math.floor(cy - radius))), min(n, int(math.ceil(cy + radius)) + 1)
        ia, ib = max(0, int(math.floor(cx - radius))), min(n, int(math.ceil(cx + radius)) + 1)
        if ja >= jb or ia >= ib:
            continue
        kk = (np.arange(ka, kb) - cz)[:, None, None] ** 2
        jj = (np.arange(ja, jb) - cy)[None, :, None] ** 2
        ii = (np.arange(ia, ib) - cx)[None, None, :] ** 2
        m[ka - z0:kb - z0, ja:jb, ia:ib] |= (kk + jj + ii) < r2
    return m


def porous7(n=128, radius=6, pe=50.0, kappa_solid=1e-4, void=0.25, seed=1):
    """BASELINE configs[2]/[4]: vertex-centred n^3, h = 1/(n+1).
    A p = -div(kappa grad p) + a.grad p, a = Pe (1, .5, .25), first-order
    upwind; face kappa = harmonic mean; Dirichlet (ghost 0, face kappa =
    own kappa) on x faces, homogeneous Neumann on y/z faces (both the
    diffusion and the upwind term of that face dropped)."""
    h = 1.0 / (n + 1)
    a = pe * np.array([1.0, 0.5, 0.25])
    centres = sphere_centres(n, radius, seed, void)

    def fn(z0, z1):
        za, zb = max(0, z0 - 1), min(n, z1 + 1)
        solid = solid_mask(n, radius, centres, za, zb)
        kap = np.where(solid, kappa_solid, 1.0)
        lo = z0 - za                      # index of plane z0 inside kap
        kc = kap[lo:lo + (z1 - z0)]
        out = np.zeros((7, z1 - z0, n, n))
        diag = np.zeros_like(kc)
        ih2 = 1.0 / h**2

        def harm(p, q):
            return 2.0 * p * q / (p + q)

        # x axis (Dirichlet)
        kf = harm(kc[:, :, 1:], kc[:, :, :-1])          # face between i-1 and i, for i>=1
        out[1][:, :, 1:] = -kf * ih2 - a[0] / h
        diag[:, :, 1:] += kf * ih2 + a[0] / h
        diag[:, :, 0] += kc[:, :, 0] * ih2 + a[0] / h   # ghost at i = -1
        out[2][:, :, :-1] = -kf * ih2
        diag[:, :, :-1] += kf * ih2
        diag[:, :, -1] += kc[:, :, -1] * ih2             # ghost at i = n
        # y axis (Neumann)
        kf = harm(kc[:, 1:, :], kc[:, :-1, :])
        out[3][:, 1:, :] = -kf * ih2 - a[1] / h
        diag[:, 1:, :] += kf * ih2 + a[1] / h
        out[4][:, :-1, :] = -kf * ih2
        diag[:, :-1, :] += kf * ih2
        # z axis (Neumann), neighbours may live in the extra planes
        for kk in range(z1 - z0):
            g = z0 + kk
            if g > 0:
                kf = harm(kc[kk], kap[lo + kk - 1])
                out[5][kk] = -kf * ih2 - a[2] / h
                diag[kk] += kf * ih2 + a[2] / h
            if g < n - 1:
                kf = harm(kc[kk], kap[lo + kk + 1])
                out[6][kk] = -kf * ih2
                diag[kk] += kf * ih2
        out[0] = diag
        return out

    return StencilProblem(
        name=f"porous{n}r{radius}", nx=n, ny=n, nz=n, periodic=0,
        offsets=OFFSETS7.copy(), _band_fn=fn, rhs_kind="sequence",
        info={"h": h, "a": a.tolist(), "radius": radius, "spheres": len(centres),
              "kappa_solid": kappa_solid},
    )


def void_fraction(prob):
    """Achieved void (fluid) fraction of a porous7 problem (reported, §8(d))."""
    n = prob.nx
    centres = sphere_centres(n, prob.info["radius"])
    fluid = 0
    step = max(1, (1 << 22) // (n * n))
    for z0 in range(0, n, step):
        z1 = min(n, z0 + step)
        fluid += int((~solid_mask(n, prob.info["radius"], centres, z0, z1)).sum())
    return fluid / prob.N
