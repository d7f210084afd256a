"""Shared check of rBiCGStab iteration scalars (tests/gpu/test_gpu_trace.py,
test_gpu_prefix.py)."""
import numpy as np

TOL = 1e-12


def check_bicg(bi, oit, r0):
    """Iteration i's scalars to (i + 1) 1e-12 (reading R21: each iteration's
    kernels contribute their 1e-12; the two trajectories then carry every
    earlier iteration's rounding difference forward)."""
    for it, (o, g) in enumerate(zip(oit, bi)):
        tol = TOL * (it + 1)
        rho, sigma, ss, ts, tt, rr = g
        rn = r0 if it == 0 else np.sqrt(oit[it - 1]["rr"])
        assert abs(rho - o["rho"]) <= tol * r0 * rn, it
        assert abs(sigma - o["sigma"]) <= tol * r0 * np.sqrt(o["vv"]), it
        assert abs(ss - o["ss"]) <= tol * o["ss"], it
        assert abs(ts - o["ts"]) <= tol * np.sqrt(o["ss"] * o["tt"]), it
        assert abs(tt - o["tt"]) <= tol * o["tt"], it
        assert abs(rr - o["rr"]) <= tol * o["rr"], it
