"""Thin Python binding of librk (include/rk.h).

PyTorch is used only for device memory, streams and process groups: every
numeric step of the solvers runs in librk's sm_100a kernels behind the
C-ABI.  The objects mirror the ABI one to one:

  Context       rk_ctx_create / rk_launch_count / rk_comm_count / rk_profile_*
  GridOperator  rk_op_create / rk_op_apply / rk_precond_apply / rk_op_update_bands
  Solver        rk_solver_create / rk_solve / rk_solve_host(_ex) / rk_solver_set_method /
                rk_recycle_set / rk_recycle_dim / rk_recycle_export / rk_history
  solve_sequence  the hybrid/sequence controller of PAPER P:662-669 (host
                  control only: switch, epoch refresh, one rk_solve per system)
"""
import ctypes as C

import numpy as np
import torch

from . import _lib as L


def _p(t):
    """Device (or host) pointer of a contiguous float64 tensor."""
    if t is None:
        return None
    assert t.is_contiguous() and t.dtype == torch.float64, "need contiguous float64"
    return C.c_void_p(t.data_ptr())


class Context:
    def __init__(self, device=0, rank=0, nranks=1, uid=None, stream=None):
        lib = L.lib()
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        h = C.c_void_p()
        L.check(lib.rk_ctx_create(device, rank, nranks, uid, C.c_void_p(stream), C.byref(h)),
                "rk_ctx_create")
        self.h = h
        self.rank, self.nranks = rank, nranks

    def launches(self):
        n = C.c_int64()
        L.check(L.lib().rk_launch_count(self.h, C.byref(n)), "rk_launch_count")
        return n.value

    def comm_count(self):
        """(all-reduce launches, halo launches) issued so far (0, 0 on one rank)."""
        a, h = C.c_int64(), C.c_int64()
        L.check(L.lib().rk_comm_count(self.h, C.byref(a), C.byref(h)), "rk_comm_count")
        return a.value, h.value

    def profile(self, on=True, filter=None, every=1):
        L.check(L.lib().rk_profile_enable(self.h, 1 if on else 0,
                                          filter.encode() if filter else None), "rk_profile_enable")
        L.check(L.lib().rk_profile_every(self.h, every), "rk_profile_every")

    def profile_read(self, reset=False):
        cap = 64
        names = C.create_string_buffer(32 * cap)
        la = (C.c_int64 * cap)()
        ms = (C.c_double * cap)()
        by = (C.c_double * cap)()
        n = C.c_int()
        L.check(L.lib().rk_profile_read(self.h, -1 if reset else cap, names, la, ms, by, C.byref(n)),
                "rk_profile_read")
        out = {}
        for i in range(min(n.value, cap)):
            nm = names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode()
            out[nm] = {"launches": la[i], "ms": ms[i], "bytes": by[i]}
        return out

    def close(self):
        if getattr(self, "h", None):
            L.lib().rk_ctx_destroy(self.h)
            self.h = None


def nccl_unique_id():
    buf = C.create_string_buffer(128)
    L.check(L.lib().rk_nccl_unique_id(buf), "rk_nccl_unique_id")
    return buf.raw


class GridOperator:
    """A in banded storage.  bands: float64 device tensor [S, nz_local, ny, nx];
    offsets: int8 [S, 3] (dx, dy, dz)."""

    def __init__(self, ctx, nx, ny, nz_global, offsets, bands, periodic=0, z0=0, nz_local=None):
        nz_local = nz_global if nz_local is None else nz_local
        self.ctx = ctx
        self.nx, self.ny, self.nz_global, self.z0, self.nz_local = nx, ny, nz_global, z0, nz_local
        self.N = nx * ny * nz_local
        self.offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.int8).reshape(-1, 3))
        g = L.rk_grid(nx, ny, nz_global, z0, nz_local, periodic)
        bands = bands.contiguous()
        assert bands.numel() == len(self.offsets) * self.N
        h = C.c_void_p()
        L.check(L.lib().rk_op_create(ctx.h, C.byref(g), len(self.offsets),
                                     self.offsets.ctypes.data_as(C.c_void_p), _p(bands), C.byref(h)),
                "rk_op_create")
        self.h = h

    def update_bands(self, bands):
        L.check(L.lib().rk_op_update_bands(self.h, _p(bands.contiguous())), "rk_op_update_bands")

    def apply(self, x, y=None):
        y = torch.empty_like(x) if y is None else y
        L.check(L.lib().rk_op_apply(self.h, _p(x), _p(y)), "rk_op_apply")
        return y

    def precond(self, r, z=None, kind=1, sweeps=5, omega_l=0.8, omega_g=1.0, zblocks=1):
        """M^-1 r: kind 1 = Jacobi(sweeps)+1 (zblocks > 1: block Jacobi, R17),
        2 = multicolour SSOR(sweeps)+1 with omega_l as the SOR relaxation (R18)."""
        z = torch.empty_like(r) if z is None else z
        pc = L.rk_precond(kind, sweeps, omega_l, omega_g, zblocks)
        L.check(L.lib().rk_precond_apply(self.h, C.byref(pc), _p(r), _p(z)), "rk_precond_apply")
        return z

    def close(self):
        if getattr(self, "h", None):
            L.lib().rk_op_destroy(self.h)
            self.h = None


def make_config(method="rgcrot", m=20, k_max=10, k_keep=5, select_count=1, precond="jacobi",
                sweeps=5, omega_l=0.8, omega_g=1.0, tol=1e-8, max_matvecs=2000,
                divergence=1e4, trunc="T1", zblocks=1, ortho="cgs2g"):
    pc = L.rk_precond({"none": 0, "jacobi": 1, "ssor": 2}[precond], sweeps, omega_l, omega_g, zblocks)
    return L.rk_config(L.METHODS[method], m, k_max, k_keep, select_count,
                       {"cgs2": 0, "cgs2g": 1}[ortho], {"T1": 0, "T2": 1}[trunc], pc, tol,
                       max_matvecs, divergence)


def config_from_params(prm, method=None, ortho="cgs2g"):
    """rk_config from any object with SolverParams-like attributes.  The
    Arnoldi orthogonalisation is librk's own choice (`ortho`: the
    Gram-corrected CGS2 of R19 by default, or "cgs2"); prm.ortho names the
    oracle's scheme and is not used here."""
    meth = method or prm.method
    if meth == "hybrid":
        meth = "rgcrot"
    k = 0 if meth in ("gmres", "bicgstab") else prm.k_max
    pcn = getattr(prm, "precond", "jacobi")
    return make_config(method=meth, m=prm.m, k_max=k, k_keep=min(prm.k_t, k),
                       select_count=0 if k == 0 else prm.p1, precond=pcn, sweeps=prm.sweeps,
                       omega_l=getattr(prm, "omega_s", 1.0) if pcn == "ssor" else prm.omega_l,
                       omega_g=prm.omega_g,
                       tol=prm.tol, max_matvecs=prm.max_mv, divergence=prm.divergence,
                       trunc=getattr(prm, "trunc", "T1"), zblocks=getattr(prm, "zblocks", 1),
                       ortho=ortho)


def _report(r):
    return {
        "outcome": L.OUTCOME_NAMES[r.outcome], "k_after": r.k_after,
        "krylov_matvecs": r.krylov_matvecs, "operator_applications": r.operator_applications,
        "cycles_or_iters": r.cycles_or_iters, "bnorm": r.bnorm,
        "final_true_res": r.final_true_res, "final_updated_res": r.final_updated_res,
        "seconds": r.seconds, "history_len": r.history_len,
    }


class Solver:
    def __init__(self, op, config):
        self.op = op
        self.config = config
        h = C.c_void_p()
        L.check(L.lib().rk_solver_create(op.h, C.byref(config), C.byref(h)), "rk_solver_create")
        self.h = h

    def set_method(self, method):
        L.check(L.lib().rk_solver_set_method(self.h, L.METHODS[method]), "rk_solver_set_method")

    def solve(self, b, x=None, tol=0.0):
        x = torch.zeros_like(b) if x is None else x
        rep = L.rk_report()
        L.check(L.lib().rk_solve(self.h, _p(b), _p(x), tol, C.byref(rep)), "rk_solve")
        return x, _report(rep)

    def solve_host(self, b_host, x_host, tol=0.0, x0_zero=False):
        """b_host, x_host: CPU float64 tensors (pinned for async copies).
        x_host holds x0 on entry unless x0_zero (x0 = 0 without touching it)."""
        rep = L.rk_report()
        L.check(L.lib().rk_solve_host_ex(self.h, _p(b_host), None if x0_zero else _p(x_host),
                                         _p(x_host), tol, C.byref(rep)), "rk_solve_host_ex")
        return x_host, _report(rep)

    def stage_rhs(self, slot, b_host):
        """Queue the upload of b_host (pinned CPU float64) into staging slot 0/1."""
        L.check(L.lib().rk_stage_rhs(self.h, slot, _p(b_host)), "rk_stage_rhs")

    def solve_staged(self, slot, x_host, tol=0.0):
        """Solve with the right-hand side staged in `slot` (x0 = 0); the download
        of x into x_host (pinned) is queued, complete after host_sync()."""
        rep = L.rk_report()
        L.check(L.lib().rk_solve_staged(self.h, slot, _p(x_host), tol, C.byref(rep)), "rk_solve_staged")
        return x_host, _report(rep)

    def host_sync(self):
        L.check(L.lib().rk_host_sync(self.h), "rk_host_sync")

    def recycle_dim(self):
        k = C.c_int()
        L.check(L.lib().rk_recycle_dim(self.h, C.byref(k)), "rk_recycle_dim")
        return k.value

    def recycle_set(self, U, C_=None, R=None):
        """U, C: device float64 [k, N] (column c = row c); R: host [k, k] or None."""
        k = 0 if U is None else U.shape[0]
        Rh = None
        if R is not None:
            Rh = np.asfortranarray(np.asarray(R, dtype=np.float64))
        L.check(L.lib().rk_recycle_set(self.h, k, _p(U) if k else None,
                                       _p(C_) if C_ is not None else None,
                                       Rh.ctypes.data_as(C.c_void_p) if Rh is not None else None,
                                       self.op.N), "rk_recycle_set")

    def recycle_export(self):
        k = self.recycle_dim()
        dev = torch.device("cuda", self.op.ctx.device)
        U = torch.empty((k, self.op.N), dtype=torch.float64, device=dev)
        Cm = torch.empty((k, self.op.N), dtype=torch.float64, device=dev)
        R = np.zeros((k, k))
        L.check(L.lib().rk_recycle_export(self.h, _p(U) if k else None, _p(Cm) if k else None,
                                          R.ctypes.data_as(C.c_void_p) if k else None,
                                          self.op.N), "rk_recycle_export")
        return U, Cm, R

    def history(self):
        n = C.c_int64()
        L.check(L.lib().rk_history(self.h, None, 0, C.byref(n)), "rk_history")
        out = np.zeros((n.value, 3))
        L.check(L.lib().rk_history(self.h, out.ctypes.data_as(C.c_void_p), n.value, C.byref(n)),
                "rk_history")
        return out

    def trace(self):
        """Per-step trace of the last solve (rk_trace): a list of rGCROT cycle
        dicts (k, m_eff, rho, lsres, H, B, y) and an [iterations x 6] array of
        rBiCGStab scalars (rho, sigma, ss, ts, tt, rr_next)."""
        out = []
        for what in (0, 1):
            n = C.c_int64()
            L.check(L.lib().rk_trace(self.h, what, None, 0, C.byref(n)), "rk_trace")
            buf = np.zeros(n.value)
            L.check(L.lib().rk_trace(self.h, what, buf.ctypes.data_as(C.c_void_p), n.value,
                                     C.byref(n)), "rk_trace")
            out.append(buf)
        cyc, pos = [], 0
        v = out[0]
        while pos < len(v):
            k, m = int(v[pos]), int(v[pos + 1])
            rho, lsres = v[pos + 2], v[pos + 3]
            pos += 4
            H = v[pos:pos + (m + 1) * m].reshape(m, m + 1).T.copy()
            pos += (m + 1) * m
            B = v[pos:pos + k * m].reshape(m, k).T.copy()
            pos += k * m
            y = v[pos:pos + m].copy()
            pos += m
            cyc.append({"k": k, "m_eff": m, "rho": rho, "lsres": lsres, "H": H, "B": B, "y": y})
        return cyc, out[1].reshape(-1, 6)

    def workspace(self):
        n = C.c_int64()
        L.check(L.lib().rk_solver_workspace(self.h, C.byref(n)), "rk_solver_workspace")
        return n.value

    def close(self):
        if getattr(self, "h", None):
            L.lib().rk_solver_destroy(self.h)
            self.h = None


def solve_sequence(solver, rhs, n, method, n_sw=0, epoch_of=None, bands_for_epoch=None,
                   tol=0.0, host=False, x_out=None, switchback=False, refresh_on_epoch=False,
                   refresh_every=0, pipeline=True, start=0, cur_epoch=None):
    """Sequence controller (reading D3): for the hybrid,
    systems t < n_sw use rGCROT and later ones rBiCGStab with the recycle
    space frozen; a new A epoch uploads its bands (librk then invalidates C
    and rebuilds it by QR of op(U) in the next solve).  Policy options
    (reading R16): `switchback` re-solves a non-converged
    rBiCGStab system by rGCROT; `refresh_on_epoch` solves the first system
    of each new A epoch after the switch by rGCROT ("intermittent solves");
    `refresh_every` = n solves every n-th post-switch system by rGCROT.
    rhs(t) -> b_t (device tensor, or pinned host tensor if host=True).
    Systems start .. start + n - 1 are solved (a sequence can be continued
    call by call: the solver keeps its recycle space).  Returns the reports;
    the solution of system start + i goes to x_out[i] when given.  The
    operator must hold the bands of epoch `cur_epoch` on entry (default: the
    epoch of system start - 1, or of system 0).  host=True with pipeline:
    b_{t+1} is uploaded and x_{t-1} downloaded while system t solves
    (rk_stage_rhs / rk_solve_staged / rk_host_sync); every x_out[i] is
    complete on return."""
    if cur_epoch is None:
        cur_epoch = (epoch_of(max(0, start - 1)) if epoch_of else 0)
    if host and pipeline:
        return _solve_sequence_pipelined(solver, rhs, n, method, n_sw, epoch_of, bands_for_epoch, tol,
                                         x_out, switchback, refresh_on_epoch, refresh_every, start,
                                         cur_epoch)
    reps = []
    cur = cur_epoch
    for i, t in enumerate(range(start, start + n)):
        e = epoch_of(t) if epoch_of else 0
        changed = e != cur
        if changed:
            solver.op.update_bands(bands_for_epoch(e))
            cur = e
        tag = method
        if method == "hybrid":
            tag = "rgcrot" if _hybrid_uses_rgcrot(t, n_sw, changed, refresh_on_epoch,
                                                  refresh_every) else "rbicgstab"
            solver.set_method(tag)
        b = rhs(t)
        x = x_out[i] if x_out is not None else torch.zeros_like(b)
        if host:   # x_hat = 0 without clearing the host buffer
            solve = lambda b_, x_: solver.solve_host(b_, x_, tol, x0_zero=True)
        else:
            x.zero_()
            solve = lambda b_, x_: solver.solve(b_, x_, tol)
        _, r = solve(b, x)
        if method == "hybrid" and tag == "rbicgstab" and switchback and r["outcome"] != "CONVERGED":
            solver.set_method("rgcrot")
            if not host:
                x.zero_()
            _, r2 = solve(b, x)
            for key in ("krylov_matvecs", "operator_applications", "seconds"):
                r2[key] += r[key]
            r = r2
            tag = "rbicgstab+rgcrot"
        r["tag"] = tag
        reps.append(r)
    return reps


def _solve_sequence_pipelined(solver, rhs, n, method, n_sw, epoch_of, bands_for_epoch, tol, x_out,
                              switchback, refresh_on_epoch, refresh_every, start=0, cur_epoch=0):
    """solve_sequence(host=True): the same controller over staged slots."""
    reps = []
    cur = cur_epoch
    bs = [rhs(start)] if n else []
    xs = []
    if n:
        solver.stage_rhs(0, bs[0])
    for i, t in enumerate(range(start, start + n)):
        if i + 1 < n:   # upload b_{t+1} while t solves
            bs.append(rhs(t + 1))
            solver.stage_rhs((i + 1) % 2, bs[i + 1])
        e = epoch_of(t) if epoch_of else 0
        changed = e != cur
        if changed:
            solver.op.update_bands(bands_for_epoch(e))
            cur = e
        tag = method
        if method == "hybrid":
            tag = "rgcrot" if _hybrid_uses_rgcrot(t, n_sw, changed, refresh_on_epoch,
                                                  refresh_every) else "rbicgstab"
            solver.set_method(tag)
        x = x_out[i] if x_out is not None else torch.zeros(bs[i].shape, dtype=torch.float64).pin_memory()
        xs.append(x)
        _, r = solver.solve_staged(i % 2, x, tol)
        if method == "hybrid" and tag == "rbicgstab" and switchback and r["outcome"] != "CONVERGED":
            solver.set_method("rgcrot")
            _, r2 = solver.solve_staged(i % 2, x, tol)
            for key in ("krylov_matvecs", "operator_applications", "seconds"):
                r2[key] += r[key]
            r = r2
            tag = "rbicgstab+rgcrot"
        r["tag"] = tag
        reps.append(r)
    solver.host_sync()
    return reps


def _hybrid_uses_rgcrot(t, n_sw, epoch_changed, refresh_on_epoch, refresh_every):
    """Hybrid schedule (R16): rGCROT for t < n_sw, and after the
    switch on the first system of a new A epoch (refresh_on_epoch) or on
    every refresh_every-th system; rBiCGStab otherwise."""
    if t < n_sw:
        return True
    if refresh_on_epoch and epoch_changed:
        return True
    return bool(refresh_every) and (t - n_sw) % refresh_every == refresh_every - 1
