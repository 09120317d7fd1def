"""Fused NCL vector kernels on device-resident vectors (include/ncl_b200.h,
``ncl_nlp_*``): the IPM / NCL per-iteration work around the KKT solve --
KktInput formation (ipm.cpp:184-208), barrier residual with its inf-norms
(kkt.cpp:341-366), bound-dual recovery + fraction-to-boundary
(kkt.cpp:316-328, ipm.cpp:124-141), trial steps, dual clipping
(ipm.cpp:232-249) and the outer update (solver.cpp:21-41, 213-217).

Vectors are passed as integer device addresses (e.g. ``tensor.data_ptr()``
of float64 CUDA tensors); the calls run on the handle's own stream and the
reductions return host scalars.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, dp, f64, i32, ip, lib


def _v(p):
    return C.c_void_p(int(p)) if p else None


class Nlp:
    def __init__(self, nt, ns, m_eq, m, jp_ptr, jp_idx, lb, ub):
        L = lib()
        self._L = L
        _lib.require_gpu()
        self.nt, self.ns, self.m_eq, self.m = nt, ns, m_eq, m
        self.n = nt + ns
        jpp, jpi, lbv, ubv = i32(jp_ptr), i32(jp_idx), f64(lb), f64(ub)
        h = C.c_void_p()
        check(L.ncl_nlp_create(nt, ns, m_eq, m, ip(jpp), ip(jpi), dp(lbv), dp(ubv), C.byref(h)), "Nlp")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.ncl_nlp_destroy(self._h)
            self._h = None

    def sync(self):
        check(self._L.ncl_nlp_sync(self._h), "sync")

    def kkt_input(self, jval, grad, c, x, zl, zu, r, y, yk, mu, rho, sigma, rbar1, rbar2, rbar3):
        check(self._L.ncl_nlp_kkt_input(self._h, *map(_v, (jval, grad, c, x, zl, zu, r, y, yk)), float(mu),
                                        float(rho), *map(_v, (sigma, rbar1, rbar2, rbar3))), "kkt_input")

    def residual(self, jval, grad, c, r, y, yk, rho, x, zl, zu, mu, stat=0, mult=0, primal=0,
                 compl_l=0, compl_u=0):
        out = np.zeros(5)
        check(self._L.ncl_nlp_residual(self._h, *map(_v, (jval, grad, c, r, y, yk)), float(rho),
                                       *map(_v, (x, zl, zu)), float(mu),
                                       *map(_v, (stat, mult, primal, compl_l, compl_u)), dp(out)), "residual")
        return out

    def step(self, x, zl, zu, mu, dx, tau, dzl, dzu):
        out = np.zeros(3)
        check(self._L.ncl_nlp_step(self._h, _v(x), _v(zl), _v(zu), float(mu), _v(dx), float(tau), _v(dzl),
                                   _v(dzu), dp(out)), "step")
        return out

    def axpy(self, n, v, a, d, out):
        check(self._L.ncl_nlp_axpy(self._h, int(n), _v(v), float(a), _v(d), _v(out)), "axpy")

    def clip_duals(self, x, mu, zl, zu):
        check(self._L.ncl_nlp_clip_duals(self._h, _v(x), float(mu), _v(zl), _v(zu)), "clip_duals")

    def outer(self, r, yk, rho_used, update):
        out = C.c_double()
        check(self._L.ncl_nlp_outer(self._h, _v(r), _v(yk), float(rho_used), int(update), C.byref(out)),
              "outer")
        return out.value


def initial_outer_state(mu0=0.1, rho0=100.0, rho_max=1e14):
    """solver.cpp:21-29: {mu, eta, omega, rho, rho_max}"""
    s = np.zeros(5)
    lib().ncl_initial_outer_state(mu0, rho0, rho_max, dp(s))
    return s


def outer_update(state, rnorm):
    """solver.cpp:31-41 (in place on the 5 schedule scalars)"""
    s = np.ascontiguousarray(state, dtype=np.float64)
    ok = lib().ncl_outer_update(dp(s), float(rnorm))
    if s is not state:
        state[:] = s
    return bool(ok)
