"""Binding of librk's per-kernel entry points (include/rk.h, "Per-kernel
entry points"): one call per kernel family of the solvers, for per-kernel
parity tests.  Argument marshalling only -- every value is computed by the
librk kernel the solvers themselves launch; there is no fallback.

Vectors are contiguous float64 CUDA tensors; a list `Q` of such tensors is
passed as a host array of device pointers.  Scalar outputs come back as
float64 CUDA tensors.  rBiCGStab records are float64 CUDA tensors of 8
values in rk_bicg_iter order (BICG_FIELDS).
"""
import ctypes as C

import torch

from . import _lib as L
from .api import _p

BICG_FIELDS = ("rho", "rr", "sigma", "ss", "ts", "tt", "flag", "stop")


def _ptrs(ts):
    arr = (C.c_void_p * max(1, len(ts)))()
    for i, t in enumerate(ts):
        arr[i] = None if t is None else _p(t).value
    return arr


def _dev(n, like):
    return torch.zeros(n, dtype=torch.float64, device=like.device)


def block_dot(ctx, Q, w, v=None):
    """K3: (Q^T w, Q^T v or None); one read of Q when v is given."""
    out_w = _dev(len(Q), w)
    out_v = _dev(len(Q), w) if v is not None else None
    L.check(L.lib().rk_block_dot(ctx.h, len(Q), _ptrs(Q), _p(w), _p(v), w.numel(), _p(out_w),
                                 _p(out_v)), "rk_block_dot")
    return out_w, out_v


def block_update(ctx, Q, g, w, dots=()):
    """K4: w <- w - Q g in place; returns [w_new^T d for d in dots] (None = w)."""
    red = _dev(max(1, len(dots)), w)
    L.check(L.lib().rk_block_update(ctx.h, len(Q), _ptrs(Q), _p(g), _p(w), w.numel(), len(dots),
                                    _ptrs(list(dots)) if dots else None, _p(red) if dots else None),
            "rk_block_update")
    return red[:len(dots)]


def block_project(ctx, Q, w, norm=True):
    """eta = Q^T w; w <- w - Q eta in place; returns (eta, ||w_new||^2 or None)."""
    eta = _dev(len(Q), w)
    nrm2 = _dev(1, w) if norm else None
    L.check(L.lib().rk_block_project(ctx.h, len(Q), _ptrs(Q), _p(w), w.numel(), _p(eta), _p(nrm2)),
            "rk_block_project")
    return eta, nrm2


def gram_update(ctx, Q, k, g, grow, w):
    """R19: h = 2 g - G g (C block of G = I, rows i >= k from grow, stride
    80); w <- w - Q h in place; returns (h, ||w_new||^2)."""
    h = _dev(len(Q), w)
    nrm2 = _dev(1, w)
    L.check(L.lib().rk_gram_update(ctx.h, len(Q), k, _ptrs(Q), _p(g), _p(grow), _p(h), _p(w),
                                   w.numel(), _p(nrm2)), "rk_gram_update")
    return h, nrm2


def project_update(ctx, C, U, xi, r, x=None):
    """Line 1b / D20: r <- r - C xi, x <- x + U xi (x optional) in place;
    returns ||r_new||^2."""
    nrm2 = _dev(1, r)
    L.check(L.lib().rk_project_update(ctx.h, len(C), _ptrs(C), _ptrs(U) if x is not None else None,
                                      _p(xi), _p(r), _p(x), r.numel(), _p(nrm2)), "rk_project_update")
    return nrm2


def normalize(ctx, w, nrm2, nin2=None):
    """Alg. 3 line 10 in place; returns the breakdown flag tensor."""
    flag = _dev(1, w)
    L.check(L.lib().rk_normalize(ctx.h, _p(w), w.numel(), _p(nrm2), _p(nin2), _p(flag)),
            "rk_normalize")
    return flag


def lincomb(ctx, Q, coef, outs, scale, acc):
    """K5: outs[o] = scale[o] * Q coef[o] (+ outs[o] if acc[o]); coef is a
    float64 CUDA tensor [nout, ncol]."""
    nout = len(outs)
    sc = (C.c_double * nout)(*[float(s) for s in scale])
    ac = (C.c_int * nout)(*[1 if a else 0 for a in acc])
    L.check(L.lib().rk_lincomb(ctx.h, len(Q), _ptrs(Q), _p(coef.contiguous()), nout, _ptrs(outs), sc,
                               ac, outs[0].numel()), "rk_lincomb")


def rotate(ctx, Q, T, kout=None):
    """K8: Q <- Q T in place (first kout columns); T float64 CUDA [k, k]
    given row-major here and passed column-major."""
    k = len(Q)
    Tc = T.t().contiguous()
    L.check(L.lib().rk_rotate(ctx.h, k, _ptrs(Q), _p(Tc), k if kout is None else kout,
                              Q[0].numel()), "rk_rotate")


def bicg_p(op, first, r, p, v, z, omega_l, jacobi, cur, prev, thr_conv, thr_div):
    L.check(L.lib().rk_bicg_p(op.h, 1 if first else 0, _p(r), _p(p), _p(v), _p(z), omega_l,
                              1 if jacobi else 0, _p(cur), _p(prev), thr_conv, thr_div), "rk_bicg_p")


def bicg_s(op, r, v, s, z, omega_l, jacobi, cur):
    L.check(L.lib().rk_bicg_s(op.h, _p(r), _p(v), _p(s), _p(z), omega_l, 1 if jacobi else 0,
                              _p(cur)), "rk_bicg_s")


def bicg_project_s(op, Cs, v, rt, ctr, r, s, z, omega_l, jacobi, cur):
    """R20 (lines 7a + 8); returns eta = C^T v."""
    eta = _dev(len(Cs), v)
    L.check(L.lib().rk_bicg_project_s(op.h, len(Cs), _ptrs(Cs), _p(v), _p(rt), _p(ctr), _p(eta),
                                      _p(r), _p(s), _p(z), omega_l, 1 if jacobi else 0, _p(cur)),
            "rk_bicg_project_s")
    return eta


def bicg_xr(op, x, r, s, t, p_hat, s_hat, rt, cur, nxt, xi=None, eta1=None, eta2=None):
    k = 0 if xi is None else xi.numel()
    L.check(L.lib().rk_bicg_xr(op.h, _p(x), _p(r), _p(s), _p(t), _p(p_hat), _p(s_hat), _p(rt),
                               _p(cur), _p(nxt), _p(xi), _p(eta1), _p(eta2), k), "rk_bicg_xr")
