"""ctypes binding of ``libncl_b200.so`` (C ABI: include/ncl_b200.h).

The shared library is built in-tree by ``csrc/Makefile`` (sm_100a only).  There
is no CPU fallback: compute entry points fail loudly when the library or a GPU
is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# NCL_B200_LIB: another build of the same library (same-box A/B timing of two
# builds, tools/ab_lib.sh); unset, the in-tree build
LIB_PATH = os.environ.get("NCL_B200_LIB") or os.path.join(PKG, "libncl_b200.so")
CSRC = os.path.join(PKG, "csrc")

_i, _d, _p, _ll = C.c_int, C.c_double, C.c_void_p, C.c_longlong
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)


class KktOpts(C.Structure):
    """KktOptions (proj/include/ncl/kkt.hpp:27-33)."""
    _fields_ = [("pivot_eps", _d), ("max_refine", _i), ("refine_tol", _d),
                ("delta_max", _d), ("accept_tol", _d)]


class KktStats(C.Structure):
    _fields_ = [("delta", _d), ("factor_attempts", _i), ("refine_steps", _i),
                ("perturbed_pivots", _i), ("rel_residual", _d), ("ok", _i),
                ("accepted", _i)]


class KktInfo(C.Structure):
    _fields_ = [("n", _i), ("nnz", _i), ("l_nnz", _ll), ("flops", _ll), ("n_supernodes", _i),
                ("sn_height", _i), ("n_paths", _i), ("n_wide", _i), ("n_levels", _i),
                ("max_front", _i), ("npairs", _ll)]


def build(force: bool = False) -> str:
    """Compile the CUDA library for sm_100a in-tree (nvcc cross-compiles
    without a GPU)."""
    args = ["make", "-s", "-C", CSRC, "-j8"]
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(args, check=True)
    return LIB_PATH


_LIB = None

# name -> (argtypes, restype)
SIGS = {
    "ncl_last_error": ([], C.c_char_p),
    "ncl_device_count": ([], _i),
    "ncl_kkt_create": ([_i, _ip, _ip, _i, _ip, _ip, _i, _i, _i, C.POINTER(KktOpts), C.POINTER(_p)], _i),
    "ncl_kkt_destroy": ([_p], None),
    "ncl_kkt_solve": ([_p, _dp, _dp, _dp, _dp, _dp, _dp, _d, _d, _dp, _dp, _dp, C.POINTER(KktStats)], _i),
    "ncl_kkt_solve_device": ([_p, _p, _p, _p, _p, _p, _p, _d, _d, _p, _p, _p, C.POINTER(KktStats)], _i),
    "ncl_kkt_info_get": ([_p, C.POINTER(KktInfo)], _i),
    "ncl_kkt_inertia_target": ([_p, _ip], _i),
    "ncl_kkt_symbolic": ([_p, _ip, _ip, _ip], _i),
    "ncl_kkt_matrix": ([_p, _ip, _ip, _dp], _i),
    "ncl_kkt_refill": ([_p, _dp, _dp, _dp, _d, _d], _i),
    "ncl_kkt_factors": ([_p, _ip, _ip, _dp, _dp, _ip], _i),
    "ncl_kkt_last_timing": ([_p, _dp], _i),
    "ncl_kkt_set_timing": ([_p, _i], _i),
    "ncl_kkt_get_stream": ([_p, C.POINTER(_p)], _i),
    "ncl_kkt_launch_count": ([_p, C.POINTER(_ll)], _i),
    "ncl_plan_create": ([_i, _ip, _ip, _i, _ip, _ip, _i, _i, _i, C.POINTER(_p)], _i),
    "ncl_plan_destroy": ([_p], None),
    "ncl_plan_info": ([_p, C.POINTER(KktInfo)], _i),
    "ncl_plan_symbolic": ([_p, _ip, _ip, _ip], _i),
    "ncl_plan_pattern": ([_p, _ip, _ip], _i),
    "ncl_plan_check_schedule": ([_p, _i], _i),
    "ncl_plan_check_dag": ([_p, _i, C.POINTER(_d)], _i),
    "ncl_amd_full_pattern": ([_i, _ip, _ip, _ip], _i),
    "ncl_analyze_host": ([_i, _i, _ip, _ip, _ip, _ip, _ip, _ip], _i),
    "ncl_sparse_create": ([_i, _i, _ip, _ip, _dp, _ip, C.POINTER(_p)], _i),
    "ncl_sparse_destroy": ([_p], None),
    "ncl_sparse_nnz": ([_p, _ip, C.POINTER(_ll)], _i),
    "ncl_sparse_symbolic": ([_p, _ip, _ip, _ip], _i),
    "ncl_sparse_factorize": ([_p, _d, _ip], _i),
    "ncl_sparse_factors": ([_p, _ip, _ip, _dp, _dp], _i),
    "ncl_sparse_ldl_solve": ([_p, _dp, _dp], _i),
    "ncl_sparse_solve_refined": ([_p, _dp, _i, _d, _dp, _ip, _dp, _ip], _i),
    "ncl_sparse_matvec": ([_p, _dp, _dp], _i),
    "ncl_nlp_create": ([_i, _i, _i, _i, _ip, _ip, _dp, _dp, C.POINTER(_p)], _i),
    "ncl_nlp_destroy": ([_p], None),
    "ncl_nlp_sync": ([_p], _i),
    "ncl_nlp_kkt_input": ([_p] + [_p] * 9 + [_d, _d] + [_p] * 4, _i),
    "ncl_nlp_residual": ([_p] + [_p] * 6 + [_d] + [_p] * 3 + [_d] + [_p] * 5 + [_dp], _i),
    "ncl_nlp_step": ([_p, _p, _p, _p, _d, _p, _d, _p, _p, _dp], _i),
    "ncl_nlp_axpy": ([_p, _i, _p, _d, _p, _p], _i),
    "ncl_nlp_clip_duals": ([_p, _p, _d, _p, _p], _i),
    "ncl_nlp_outer": ([_p, _p, _p, _d, _i, _dp], _i),
    "ncl_initial_outer_state": ([_d, _d, _d, _dp], None),
    "ncl_init_multipliers": ([_i, _i, _i, _ip, _ip, _dp, _dp, _dp, _dp], _i),
    "ncl_jjt_candidates": ([_i, _i, _ip, _ip, _ll, C.POINTER(_ll), _ip, _ip], _i),
    "ncl_schur_create": ([_i, _ip, _ip, _i, _ip, _ip, _i, _i, _i, C.POINTER(KktOpts), C.POINTER(_p)], _i),
    "ncl_schur_destroy": ([_p], None),
    "ncl_schur_info": ([_p, C.POINTER(KktInfo)], _i),
    "ncl_schur_n0": ([_p], _i),
    "ncl_schur_factor": ([_p, _p, _p, _p, _d, _d, _ip, _p], _i),
    "ncl_schur_factor_dense": ([_p, _p, _d, _ip], _i),
    "ncl_schur_rhs": ([_p, _p, _p, _p, _p, _p, _d, _d, _p], _i),
    "ncl_schur_forward": ([_p, _p, _p], _i),
    "ncl_schur_solve0": ([_p, _p, _p], _i),
    "ncl_schur_backward": ([_p, _p, _p], _i),
    "ncl_schur_residual": ([_p, _p, _p, _p], _i),
    "ncl_schur_recover": ([_p, _p, _p, _p, _d, _d, _p, _p, _p], _i),
    "ncl_schur_launch_count": ([_p, C.POINTER(_ll)], _i),
    "ncl_outer_update": ([_dp, _d], _i),
}


def lib():
    """Load the library (building it when absent).  Raises when it cannot be
    built or loaded."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _LIB = L
    return _LIB


class NclError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().ncl_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        if rc == -2:
            raise LookupError(f"{what}: {msg}")
        raise NclError(f"{what} failed ({rc}): {msg}")


def require_gpu() -> None:
    if lib().ncl_device_count() < 1:
        raise NclError("no CUDA device visible: the sm_100a path has no CPU fallback")


def ip(a):
    return a.ctypes.data_as(_ip) if a is not None else None


def dp(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))
