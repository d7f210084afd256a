"""ctypes declarations of the librk C-ABI (include/rk.h).  Argument
marshalling only: every step of the solver runs in librk's CUDA kernels.
Loading fails loudly if librk.so is missing -- there is no fallback."""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RK_LIBPATH: an A/B variant built by scripts/build_variant.py (measurement only)
LIBPATH = os.environ.get("RK_LIBPATH") or os.path.join(HERE, "librk.so")

RK_OK, RK_EINVAL, RK_ECUDA, RK_ENCCL, RK_ENOMEM, RK_ESTATE, RK_EUNSUPPORTED = range(7)
STATUS_NAMES = ["RK_OK", "RK_EINVAL", "RK_ECUDA", "RK_ENCCL", "RK_ENOMEM", "RK_ESTATE",
                "RK_EUNSUPPORTED"]
RK_CONVERGED, RK_MAX_MATVECS, RK_BREAKDOWN, RK_STAGNATION, RK_UNSTABLE, RK_DRIFT = range(6)
OUTCOME_NAMES = ["CONVERGED", "MAX_MATVECS", "BREAKDOWN", "STAGNATION", "UNSTABLE", "DRIFT"]
RK_GMRES, RK_RGCROT, RK_BICGSTAB, RK_RBICGSTAB = range(4)
METHODS = {"gmres": RK_GMRES, "rgcrot": RK_RGCROT, "bicgstab": RK_BICGSTAB,
           "rbicgstab": RK_RBICGSTAB}


class rk_grid(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz_global", C.c_int64),
                ("z0", C.c_int64), ("nz_local", C.c_int64), ("periodic_mask", C.c_uint32)]


class rk_precond(C.Structure):
    _fields_ = [("kind", C.c_int), ("sweeps", C.c_int), ("omega_local", C.c_double),
                ("omega_global", C.c_double), ("zblocks", C.c_int)]


class rk_config(C.Structure):
    _fields_ = [("method", C.c_int), ("m", C.c_int), ("k_max", C.c_int), ("k_keep", C.c_int),
                ("select_count", C.c_int), ("ortho", C.c_int), ("trunc", C.c_int),
                ("pc", rk_precond), ("tol", C.c_double), ("max_matvecs", C.c_int64),
                ("divergence_factor", C.c_double)]


class rk_report(C.Structure):
    _fields_ = [("outcome", C.c_int32), ("k_after", C.c_int32), ("krylov_matvecs", C.c_int64),
                ("operator_applications", C.c_int64), ("cycles_or_iters", C.c_int64),
                ("bnorm", C.c_double), ("final_true_res", C.c_double),
                ("final_updated_res", C.c_double), ("seconds", C.c_double),
                ("history_len", C.c_int64)]


class RkError(RuntimeError):
    pass


_lib = None


def lib():
    """Load librk.so (built in-tree by paper_1501_03358_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIBPATH):
        raise RkError(f"librk.so not found at {LIBPATH}: run `python -m paper_1501_03358_b200.build` "
                      "(there is no CPU fallback)")
    L = C.CDLL(LIBPATH)
    vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
    P = C.POINTER
    sig = {
        "rk_last_error": ([], C.c_char_p),
        "rk_version": ([], C.c_char_p),
        "rk_nccl_unique_id": ([C.c_char_p], i32),
        "rk_ctx_create": ([i32, i32, i32, C.c_char_p, vp, P(vp)], i32),
        "rk_ctx_destroy": ([vp], None),
        "rk_op_create": ([vp, P(rk_grid), i32, vp, vp, P(vp)], i32),
        "rk_op_update_bands": ([vp, vp], i32),
        "rk_op_destroy": ([vp], None),
        "rk_op_apply": ([vp, vp, vp], i32),
        "rk_precond_apply": ([vp, P(rk_precond), vp, vp], i32),
        "rk_solver_create": ([vp, P(rk_config), P(vp)], i32),
        "rk_solver_destroy": ([vp], None),
        "rk_solver_set_method": ([vp, i32], i32),
        "rk_recycle_set": ([vp, i32, vp, vp, vp, i64], i32),
        "rk_recycle_dim": ([vp, P(i32)], i32),
        "rk_recycle_export": ([vp, vp, vp, vp, i64], i32),
        "rk_solve": ([vp, vp, vp, dbl, P(rk_report)], i32),
        "rk_solve_host": ([vp, vp, vp, dbl, P(rk_report)], i32),
        "rk_solve_host_ex": ([vp, vp, vp, vp, dbl, P(rk_report)], i32),
        "rk_stage_rhs": ([vp, i32, vp], i32),
        "rk_solve_staged": ([vp, i32, vp, dbl, P(rk_report)], i32),
        "rk_host_sync": ([vp], i32),
        "rk_history": ([vp, vp, i64, P(i64)], i32),
        "rk_trace": ([vp, i32, vp, i64, P(i64)], i32),
        "rk_solver_workspace": ([vp, P(i64)], i32),
        "rk_launch_count": ([vp, P(i64)], i32),
        "rk_comm_count": ([vp, P(i64), P(i64)], i32),
        "rk_profile_enable": ([vp, i32, C.c_char_p], i32),
        "rk_profile_every": ([vp, i32], i32),
        "rk_profile_read": ([vp, i32, vp, vp, vp, vp, P(i32)], i32),
        # per-kernel entry points (pointer arrays are passed as c_void_p)
        "rk_block_dot": ([vp, i32, vp, vp, vp, i64, vp, vp], i32),
        "rk_block_update": ([vp, i32, vp, vp, vp, i64, i32, vp, vp], i32),
        "rk_block_project": ([vp, i32, vp, vp, i64, vp, vp], i32),
        "rk_gram_update": ([vp, i32, i32, vp, vp, vp, vp, vp, i64, vp], i32),
        "rk_project_update": ([vp, i32, vp, vp, vp, vp, vp, i64, vp], i32),
        "rk_normalize": ([vp, vp, i64, vp, vp, vp], i32),
        "rk_lincomb": ([vp, i32, vp, vp, i32, vp, vp, vp, i64], i32),
        "rk_rotate": ([vp, i32, vp, vp, i32, i64], i32),
        "rk_bicg_p": ([vp, i32, vp, vp, vp, vp, dbl, i32, vp, vp, dbl, dbl], i32),
        "rk_bicg_s": ([vp, vp, vp, vp, vp, dbl, i32, vp], i32),
        "rk_bicg_project_s": ([vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, dbl, i32, vp], i32),
        "rk_bicg_xr": ([vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def check(status, what=""):
    if status != RK_OK:
        msg = lib().rk_last_error().decode(errors="replace")
        raise RkError(f"{what}: {STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")


# Every symbol include/rk.h declares (checked by the CPU test suite).
EXPORTED = ["rk_last_error", "rk_version", "rk_nccl_unique_id", "rk_ctx_create",
            "rk_ctx_destroy", "rk_op_create", "rk_op_update_bands", "rk_op_destroy",
            "rk_op_apply", "rk_precond_apply", "rk_solver_create", "rk_solver_destroy",
            "rk_solver_set_method", "rk_recycle_set", "rk_recycle_dim", "rk_recycle_export",
            "rk_solve", "rk_solve_host", "rk_solve_host_ex", "rk_stage_rhs", "rk_solve_staged",
            "rk_host_sync", "rk_history", "rk_trace", "rk_solver_workspace", "rk_launch_count",
            "rk_comm_count",
            "rk_profile_enable", "rk_profile_every", "rk_profile_read",
            "rk_block_dot", "rk_block_update", "rk_block_project", "rk_gram_update", "rk_project_update",
            "rk_normalize", "rk_lincomb", "rk_rotate", "rk_bicg_p", "rk_bicg_s",
            "rk_bicg_project_s", "rk_bicg_xr"]
