"""Multi-rank (z-slab) decomposition on CPU with torch.distributed/gloo.

librk's multi-GPU path (comm.cpp) keeps one ghost plane below and above every
rank's slab, fills them before every stencil application by exchanging
planes with the z-neighbours -- first every rank sends its TOP plane up and
receives its lower ghost from below, then sends its BOTTOM plane down and
receives its upper ghost from above (periodic z: a ring) -- and sums every
batch of partial dot products with one all-reduce, so the tiny Krylov state
(H, B, alpha, ...) is replicated bit-identically.  librk's OWN schedule of
those calls runs at world 2/3 in tests/gpu/test_gpu_multirank.py (an
in-process rank group on one GPU); here, without a GPU, the same protocol
runs with gloo over world_size 2 and 3 and is checked against the
single-domain oracle:
  * halo exchange + local stencil == global SpMV (periodic and Dirichlet z),
  * the Jacobi(5+1) preconditioner with a halo per sweep == global M^-1,
  * block Jacobi with one z-block per rank and NO halo in the local sweeps
    == the oracle's global block-Jacobi M^-1 (reading R17),
  * one GMRES cycle with all-reduced (batched, CGS2) dots == the global one,
  * the reduced scalars are bit-identical on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.krylov import gmres
from oracle.stencil import Jacobi, Operator, shifted
from problems import SolverParams, get_workload, slab_range
from problems.stencils import channel19, porous7


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ------------------------------------------------------------ slab emulation
class Slab:
    """One rank's slab: bands [S, nzl, ny, nx], padded vectors [nzl + 2, ny, nx]."""

    def __init__(self, prob, rank, world):
        self.prob, self.rank, self.world = prob, rank, world
        self.z0, self.z1 = slab_range(prob.nz, rank, world)
        self.nzl = self.z1 - self.z0
        self.bands = prob.bands(self.z0, self.z1)
        self.offsets = prob.offsets
        self.pz = bool(prob.periodic & 4)

    def pad(self, v):
        out = np.zeros((self.nzl + 2, self.prob.ny, self.prob.nx))
        out[1:-1] = v.reshape(self.nzl, self.prob.ny, self.prob.nx)
        return out

    def halo(self, xp):
        """comm.cpp::halo with gloo: up-then-down, matched in issue order."""
        R, me = self.world, self.rank
        up, dn = me + 1, me - 1
        if self.pz:
            up %= R
            dn = (dn + R) % R
        else:
            up = up if up < R else -1
        reqs = []
        top = torch.from_numpy(xp[-2].copy())
        bot = torch.from_numpy(xp[1].copy())
        glo = torch.zeros_like(top)
        ghi = torch.zeros_like(top)
        # the four operations in comm.cpp's order; isend/irecv keep gloo from blocking
        if up >= 0:
            reqs.append(dist.isend(top, up))
        if dn >= 0:
            reqs.append(dist.irecv(glo, dn))
        if dn >= 0:
            reqs.append(dist.isend(bot, dn))
        if up >= 0:
            reqs.append(dist.irecv(ghi, up))
        for r in reqs:
            r.wait()
        xp[0] = glo.numpy() if dn >= 0 else 0.0
        xp[-1] = ghi.numpy() if up >= 0 else 0.0

    def spmv(self, v):
        """halo exchange, then the local stencil (x/y wrap per mask, z from ghosts)."""
        xp = self.pad(v)
        self.halo(xp)
        y = np.zeros((self.nzl, self.prob.ny, self.prob.nx))
        mask_xy = self.prob.periodic & 3          # z handled by the ghost planes
        for d, (dx, dy, dz) in enumerate(self.offsets):
            xs = shifted(xp, int(dx), int(dy), 0, mask_xy)[1 + dz:1 + dz + self.nzl]
            y += self.bands[d] * xs
        return y.reshape(-1)

    def jacobi(self, r, sweeps=5, wl=0.8, wg=1.0):
        D = self.bands[0].reshape(-1)
        z = wl * r / D
        for _ in range(sweeps - 1):
            z = z + wl * (r - self.spmv(z)) / D
        return z + wg * (r - self.spmv(z)) / D

    def spmv_local(self, v):
        """Local stencil with zero ghost planes and NO exchange: the operator
        of the block-Jacobi local sweeps when every rank owns one z-block
        (reading R17; librk skips the halo for such sweeps)."""
        xp = self.pad(v)
        y = np.zeros((self.nzl, self.prob.ny, self.prob.nx))
        mask_xy = self.prob.periodic & 3
        for d, (dx, dy, dz) in enumerate(self.offsets):
            xs = shifted(xp, int(dx), int(dy), 0, mask_xy)[1 + dz:1 + dz + self.nzl]
            y += self.bands[d] * xs
        return y.reshape(-1)

    def block_jacobi(self, r, sweeps=5, wl=0.8, wg=1.0):
        D = self.bands[0].reshape(-1)
        z = wl * r / D
        for _ in range(sweeps - 1):
            z = z + wl * (r - self.spmv_local(z)) / D
        return z + wg * (r - self.spmv(z)) / D

    def allreduce(self, vals):
        t = torch.tensor(np.asarray(vals, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()


def dist_gmres_cycle(sl, b, m):
    """One left-preconditioned GMRES(m) cycle (Alg. 1) from x0 = 0, with CGS2
    (reading D8) and one all-reduce per batch of dots, as librk batches them."""
    r = sl.jacobi(b)
    rho = np.sqrt(sl.allreduce([r @ r])[0])
    V = [r / rho]
    H = np.zeros((m + 1, m))
    for j in range(m):
        w = sl.jacobi(sl.spmv(V[j]))
        Q = np.stack(V)
        for _ in range(2):
            g = sl.allreduce(Q @ w)
            w = w - g @ Q
            H[:j + 1, j] += g
        H[j + 1, j] = np.sqrt(sl.allreduce([w @ w])[0])
        V.append(w / H[j + 1, j])
    e1 = np.zeros(m + 1)
    e1[0] = rho
    y = np.linalg.lstsq(H, e1, rcond=None)[0]
    return np.stack(V[:m]).T @ y, H


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = {"channel": lambda: channel19(12), "porous": lambda: porous7(12, 2)}[case]()
        sl = Slab(prob, rank, world)
        rng = np.random.default_rng(7)
        xg = rng.uniform(-1, 1, prob.N)
        P = prob.nx * prob.ny
        xl = xg[sl.z0 * P:sl.z1 * P]
        y = sl.spmv(xl)
        z = sl.jacobi(xl)
        zbj = sl.block_jacobi(xl)
        b = prob.rhs(1, sl.z0, sl.z1).reshape(-1)
        xc, H = dist_gmres_cycle(sl, b, 6)
        # replicated state must be bit-identical across ranks
        Ht = torch.from_numpy(H.copy())
        Hs = [torch.zeros_like(Ht) for _ in range(world)]
        dist.all_gather(Hs, Ht)
        same = all(torch.equal(Hs[0], h) for h in Hs)
        q.put((rank, sl.z0, sl.z1, y, z, zbj, xc, same))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["channel", "porous"])
@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_matches_global(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    prob = {"channel": lambda: channel19(12), "porous": lambda: porous7(12, 2)}[case]()
    op = Operator.from_problem(prob)
    pc = Jacobi(op)
    xg = np.random.default_rng(7).uniform(-1, 1, prob.N)
    yg = op.apply(xg)
    zg = pc(xg)
    b = prob.rhs(1).reshape(-1)
    xc_g, _ = gmres(op, pc, b, SolverParams(m=6, k_max=0, p1=0, tol=1e-30, max_mv=6))
    zbj_g = Jacobi(op, zblocks=world)(xg) if prob.nz % world == 0 else None
    P = prob.nx * prob.ny
    for rank, z0, z1, y, z, zbj, xc, same in res:
        sl = slice(z0 * P, z1 * P)
        assert np.allclose(y, yg[sl], rtol=0, atol=1e-12 * np.abs(yg).max())
        assert np.allclose(z, zg[sl], rtol=0, atol=1e-12 * np.abs(zg).max())
        if zbj_g is not None:     # halo-free local sweeps == global block Jacobi (R17)
            assert np.allclose(zbj, zbj_g[sl], rtol=0, atol=1e-12 * np.abs(zbj_g).max())
        assert np.allclose(xc, xc_g[sl], rtol=0, atol=1e-10 * np.abs(xc_g).max())
        assert same, "replicated Hessenberg differs across ranks"
