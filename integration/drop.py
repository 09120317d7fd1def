"""ctypes front of the drop-in build (integration/_build/libncl_drop.so): the
reference's own NCL outer loop and IPM driver (proj/src/solver.cpp, ipm.cpp,
model.cpp, compiled unmodified) running on the B200 KktContext
(integration/kkt_b200.cpp -> include/ncl_b200.h).

    from integration.drop import DropModel
    rep = DropModel("opf_mesh:40:40:1").solve(form="k1s", tol=1e-8)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libncl_drop.so")

_i, _d, _p = C.c_int, C.c_double, C.c_void_p
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)
FORMS = {"k2": 0, "k2r": 1, "k1s": 2}
STATUS = ["optimal", "infeasible", "iteration_limit", "numeric_error"]

_L = None


def available() -> bool:
    return os.path.exists(LIB)


def build() -> None:
    """Needs the reference sources (/root/reference) -- this container only."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _L
    if _L is None:
        if not available():
            build()
        L = C.CDLL(LIB)
        L.drop_model_new.argtypes = [C.c_char_p]
        L.drop_model_new.restype = _p
        L.drop_model_free.argtypes = [_p]
        L.drop_model_dims.argtypes = [_p, _ip]
        L.drop_solve.argtypes = [_p, _i, _d, _i, _i, _d, _i]
        L.drop_solve.restype = _p
        L.drop_report_free.argtypes = [_p]
        L.drop_report_scalars.argtypes = [_p, _dp]
        L.drop_report_log.argtypes = [_p, _dp, _dp]
        L.drop_report_xy.argtypes = [_p, _dp, _dp]
        _L = L
    return _L


class DropModel:
    def __init__(self, spec: str):
        self.L = lib()
        self.h = self.L.drop_model_new(spec.encode())
        if not self.h:
            raise ValueError(f"unknown instance {spec}")
        d = np.zeros(6, np.int32)
        self.L.drop_model_dims(self.h, d.ctypes.data_as(_ip))
        self.nt, self.ns, self.m_eq, self.m = (int(v) for v in d[:4])
        self.n = self.nt + self.ns

    def __del__(self):
        if getattr(self, "h", None):
            self.L.drop_model_free(self.h)
            self.h = None

    def solve(self, form="k1s", tol=1e-8, max_outer=40, max_inner=1000, pivot_eps=1e-10, scaling=True):
        L = self.L
        r = L.drop_solve(self.h, FORMS[form], tol, max_outer, max_inner, pivot_eps, int(scaling))
        sc = np.zeros(12)
        L.drop_report_scalars(r, sc.ctypes.data_as(_dp))
        nlog, nex = int(sc[10]), int(sc[11])
        log = np.zeros((max(nlog, 1), 13))
        ex = np.zeros(max(nex, 1))
        L.drop_report_log(r, log.ctypes.data_as(_dp), ex.ctypes.data_as(_dp))
        x = np.zeros(self.n)
        y = np.zeros(self.m)
        L.drop_report_xy(r, x.ctypes.data_as(_dp), y.ctypes.data_as(_dp))
        L.drop_report_free(r)
        return dict(status=STATUS[int(sc[0])], outer_iters=int(sc[1]), inner_iters=int(sc[2]),
                    extrapolation_accepts=int(sc[3]), objective=sc[4], kkt_residual=sc[5],
                    primal_feas=sc[6], mu_final=sc[7], rho_final=sc[8], solve_seconds=sc[9],
                    log=log[:nlog], extrap_alpha=ex[:nex], x=x, y=y)
