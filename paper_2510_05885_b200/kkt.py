"""Host-side mirror of the reference's KKT plugin API on the B200 path.

Names, argument meaning and error behaviour follow
proj/include/ncl/kkt.hpp:22-125 and proj/include/ncl/sparse.hpp:26-99:

* ``KktContext(hp, jp, nt, ns, m_eq, form, opt)`` -- symbolic analysis once
  (kkt.cpp:41-138); ``solve(in, warm_delta) -> KktStep`` (kkt.cpp:266-314);
  ``form()``, ``inertia_target()``, ``system_size()``, ``matrix()``.
  Inconsistent shapes raise ``ValueError`` (std::invalid_argument); numerical
  failure is ``KktStep.ok == False``, never an exception.
* ``SparseLdl`` -- ``sym_from_triplets`` + ``analyze`` / ``factorize`` /
  ``ldl_solve`` / ``solve_refined`` on the device LDL^T.
* ``KktPlan`` -- the host-only symbolic half (no GPU needed).

Every compute call goes through ``libncl_b200.so``; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional

import numpy as np

from . import _lib
from ._lib import KktInfo, KktOpts, KktStats, check, dp, f64, i32, ip, lib


class KktForm(IntEnum):
    """proj/include/ncl/kkt.hpp:22"""
    K2 = 0
    K2r = 1
    K1s = 2


_FORM_NAMES = {"k2": KktForm.K2, "k2r": KktForm.K2r, "k1s": KktForm.K1s}


def parse_kkt_form(name: str) -> KktForm:
    """kkt.cpp:10-15"""
    try:
        return _FORM_NAMES[name]
    except KeyError:
        raise ValueError(f"unknown kkt form: {name}") from None


def kkt_form_name(f: KktForm) -> str:
    return {KktForm.K2: "k2", KktForm.K2r: "k2r", KktForm.K1s: "k1s"}[KktForm(f)]


@dataclass
class HessianPattern:
    """Lower-triangle CSC over the nt decision variables (model.hpp:44-48)."""
    n: int
    ptr: np.ndarray
    idx: np.ndarray

    def nnz(self) -> int:
        return int(self.ptr[-1]) if len(self.ptr) else 0


@dataclass
class JacobianPattern:
    """CSR, equality rows first, sorted columns (model.hpp:38-42)."""
    rows: int
    cols: int
    ptr: np.ndarray
    idx: np.ndarray

    def nnz(self) -> int:
        return int(self.ptr[-1]) if len(self.ptr) else 0


@dataclass
class KktOptions:
    """proj/include/ncl/kkt.hpp:27-33"""
    pivot_eps: float = 1e-10
    max_refine: int = 10
    refine_tol: float = 1e-12
    delta_max: float = 1e40
    accept_tol: float = 1e-8

    def _c(self) -> KktOpts:
        return KktOpts(self.pivot_eps, self.max_refine, self.refine_tol, self.delta_max,
                       self.accept_tol)


@dataclass
class KktInput:
    """proj/include/ncl/kkt.hpp:38-46: hval/jval follow the model patterns,
    sigma and rbar1 cover x = (t, s), rbar2/rbar3 the m rows."""
    hval: np.ndarray
    jval: np.ndarray
    sigma: np.ndarray
    rbar1: np.ndarray
    rbar2: np.ndarray
    rbar3: np.ndarray
    rho: float = 0.0


@dataclass
class KktStep:
    """proj/include/ncl/kkt.hpp:48-56"""
    dx: np.ndarray = field(default_factory=lambda: np.zeros(0))
    dr: np.ndarray = field(default_factory=lambda: np.zeros(0))
    dy: np.ndarray = field(default_factory=lambda: np.zeros(0))
    delta: float = 0.0
    factor_attempts: int = 0
    refine_steps: int = 0
    perturbed_pivots: int = 0
    rel_residual: float = 0.0
    ok: bool = False


def _shape_args(hp: HessianPattern, jp: JacobianPattern):
    return (i32(hp.ptr), i32(hp.idx), i32(jp.ptr), i32(jp.idx))


class KktPlan:
    """Host-only symbolic plan of a KKT pattern (no GPU needed)."""

    def __init__(self, hp: HessianPattern, jp: JacobianPattern, nt: int, ns: int, m_eq: int,
                 form: KktForm):
        L = lib()
        self._L = L
        hpp, hpi, jpp, jpi = _shape_args(hp, jp)
        h = C.c_void_p()
        check(L.ncl_plan_create(nt, ip(hpp), ip(hpi), jp.rows, ip(jpp), ip(jpi), ns, m_eq,
                                int(form), C.byref(h)), "KktPlan")
        self._h = h
        self.info = KktInfo()
        check(L.ncl_plan_info(h, C.byref(self.info)), "ncl_plan_info")

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.ncl_plan_destroy(self._h)
            self._h = None

    def symbolic(self):
        n = self.info.n
        perm = np.zeros(n, np.int32)
        parent = np.zeros(n, np.int32)
        lcp = np.zeros(n + 1, np.int32)
        check(self._L.ncl_plan_symbolic(self._h, ip(perm), ip(parent), ip(lcp)), "symbolic")
        return dict(perm=perm, parent=parent, lcol_ptr=lcp)

    def pattern(self):
        n, nnz = self.info.n, self.info.nnz
        cp = np.zeros(n + 1, np.int32)
        ri = np.zeros(nnz, np.int32)
        check(self._L.ncl_plan_pattern(self._h, ip(cp), ip(ri)), "pattern")
        return cp, ri


class KktContext:
    """Drop-in ``ncl::KktContext`` on the B200 (kkt.hpp:58-93)."""

    def __init__(self, hp: HessianPattern, jp: JacobianPattern, nt: int, ns: int, m_eq: int,
                 form: KktForm, opt: Optional[KktOptions] = None):
        L = lib()
        self._L = L
        _lib.require_gpu()
        self._form = KktForm(form)
        self.nt, self.ns, self.m_eq, self.m = nt, ns, m_eq, jp.rows
        self.n = nt + ns
        self.hnnz, self.jnnz = hp.nnz(), jp.nnz()
        hpp, hpi, jpp, jpi = _shape_args(hp, jp)
        h = C.c_void_p()
        o = (opt or KktOptions())._c()
        check(L.ncl_kkt_create(nt, ip(hpp), ip(hpi), jp.rows, ip(jpp), ip(jpi), ns, m_eq,
                               int(form), C.byref(o), C.byref(h)), "KktContext")
        self._h = h
        self.info = KktInfo()
        check(L.ncl_kkt_info_get(h, C.byref(self.info)), "ncl_kkt_info_get")

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.ncl_kkt_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def form(self) -> KktForm:
        return self._form

    def inertia_target(self):
        t = np.zeros(3, np.int32)
        check(self._L.ncl_kkt_inertia_target(self._h, ip(t)), "inertia_target")
        return tuple(int(v) for v in t)

    def system_size(self) -> int:
        return int(self.info.n)

    def solve(self, inp: KktInput, warm_delta: float, out=None) -> KktStep:
        """kkt.hpp:61 KktContext::solve.  out: optional caller-owned (dx, dr, dy)
        float64 arrays to receive the step (e.g. pinned host memory)."""
        hv, jv = f64(inp.hval), f64(inp.jval)
        sg, r1, r2, r3 = f64(inp.sigma), f64(inp.rbar1), f64(inp.rbar2), f64(inp.rbar3)
        if (len(hv) != self.hnnz or len(jv) != self.jnnz or len(sg) != self.n or len(r1) != self.n
                or len(r2) != self.m or len(r3) != self.m):
            raise ValueError("kkt: input lengths do not match the problem shape")
        if out is None:
            dx, dr, dy = np.zeros(self.n), np.zeros(self.m), np.zeros(self.m)
        else:
            dx, dr, dy = out
            if not all(a.dtype == np.float64 and a.flags.c_contiguous for a in out) or \
                    (len(dx), len(dr), len(dy)) != (self.n, self.m, self.m):
                raise ValueError("kkt: out must be contiguous float64 arrays of lengths (n, m, m)")
        st = KktStats()
        check(self._L.ncl_kkt_solve(self._h, dp(hv), dp(jv), dp(sg), dp(r1), dp(r2), dp(r3),
                                    float(inp.rho), float(warm_delta), dp(dx), dp(dr), dp(dy),
                                    C.byref(st)), "KktContext.solve")
        if not st.accepted:  # kkt.cpp:291-298: an accepted attempt keeps its step, finite or not
            dx, dr, dy = np.zeros(0), np.zeros(0), np.zeros(0)
        return KktStep(dx, dr, dy, st.delta, st.factor_attempts, st.refine_steps,
                       st.perturbed_pivots, st.rel_residual, bool(st.ok))

    def solve_device(self, ptrs, rho: float, warm_delta: float, out_ptrs) -> KktStats:
        """Device-pointer variant: ptrs = (hval, jval, sigma, rbar1, rbar2,
        rbar3), out_ptrs = (dx, dr, dy) as integer device addresses."""
        st = KktStats()
        check(self._L.ncl_kkt_solve_device(self._h, *[C.c_void_p(p) for p in ptrs], float(rho),
                                           float(warm_delta),
                                           *[C.c_void_p(p) for p in out_ptrs], C.byref(st)),
              "KktContext.solve_device")
        return st

    def matrix(self):
        """Pattern and values of the last refill (kkt.hpp:70)."""
        n, nnz = self.info.n, self.info.nnz
        cp = np.zeros(n + 1, np.int32)
        ri = np.zeros(nnz, np.int32)
        v = np.zeros(nnz)
        check(self._L.ncl_kkt_matrix(self._h, ip(cp), ip(ri), dp(v)), "matrix")
        return cp, ri, v

    def refill(self, inp: KktInput, delta: float) -> np.ndarray:
        check(self._L.ncl_kkt_refill(self._h, dp(f64(inp.hval)), dp(f64(inp.jval)),
                                     dp(f64(inp.sigma)), float(inp.rho), float(delta)), "refill")
        return self.matrix()[2]

    def symbolic(self):
        n = self.info.n
        perm = np.zeros(n, np.int32)
        parent = np.zeros(n, np.int32)
        lcp = np.zeros(n + 1, np.int32)
        check(self._L.ncl_kkt_symbolic(self._h, ip(perm), ip(parent), ip(lcp)), "symbolic")
        return dict(perm=perm, parent=parent, lcol_ptr=lcp)

    def factors(self):
        """Last factorization in the reference's LdlFactors layout."""
        n, lnz = self.info.n, self.info.l_nnz
        lcp = np.zeros(n + 1, np.int32)
        lri = np.zeros(lnz, np.int32)
        lv = np.zeros(lnz)
        d = np.zeros(n)
        info = np.zeros(4, np.int32)
        check(self._L.ncl_kkt_factors(self._h, ip(lcp), ip(lri), dp(lv), dp(d), ip(info)), "factors")
        return dict(ok=bool(info[0]), n_pos=int(info[1]), n_neg=int(info[2]),
                    perturbed=int(info[3]), lcol_ptr=lcp, lrow_ind=lri, lval=lv, d=d)

    def stream(self) -> int:
        """the context's cudaStream_t (for torch.cuda.ExternalStream timing)"""
        s = C.c_void_p()
        check(self._L.ncl_kkt_get_stream(self._h, C.byref(s)), "get_stream")
        return s.value or 0

    def launch_count(self) -> int:
        n = C.c_longlong()
        check(self._L.ncl_kkt_launch_count(self._h, C.byref(n)), "launch_count")
        return n.value

    def set_timing(self, on: bool = True) -> None:
        check(self._L.ncl_kkt_set_timing(self._h, int(on)), "set_timing")

    def last_timing(self):
        ms = np.zeros(6)
        check(self._L.ncl_kkt_last_timing(self._h, dp(ms)), "last_timing")
        return dict(assemble_ms=ms[0], factor_ms=ms[1], solve_ms=ms[2], recover_ms=ms[3],
                    total_ms=ms[4], solves=int(ms[5]))


def recover_bound_duals(x, lb, ub, zl, zu, mu, dx):
    """kkt.cpp:316-328 (host convenience; the device kernel lives in
    ``ncl_vec``)."""
    x, lb, ub, zl, zu, dx = map(f64, (x, lb, ub, zl, zu, dx))
    dzl = np.zeros_like(x)
    dzu = np.zeros_like(x)
    fl = np.isfinite(lb)
    fu = np.isfinite(ub)
    dzl[fl] = -(zl[fl] * dx[fl] - mu) / (x[fl] - lb[fl]) - zl[fl]
    dzu[fu] = (zu[fu] * dx[fu] + mu) / (ub[fu] - x[fu]) - zu[fu]
    return dzl, dzu


class SparseLdl:
    """sparse.hpp API on the device LDL^T: triplets (mirrored, duplicates
    summed) -> analyze (AMD, or ``perm``) -> factorize -> solves."""

    def __init__(self, n: int, rows, cols, vals, perm=None):
        L = lib()
        self._L = L
        _lib.require_gpu()
        r, c, v = i32(rows), i32(cols), f64(vals)
        pm = None if perm is None else i32(perm)
        h = C.c_void_p()
        check(L.ncl_sparse_create(n, len(r), ip(r), ip(c), dp(v), ip(pm), C.byref(h)), "SparseLdl")
        self._h = h
        self.n = n
        nnz = C.c_int()
        lnz = C.c_longlong()
        check(L.ncl_sparse_nnz(h, C.byref(nnz), C.byref(lnz)), "nnz")
        self.nnz, self.l_nnz = nnz.value, lnz.value

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.ncl_sparse_destroy(self._h)
            self._h = None

    def symbolic(self):
        n = self.n
        perm = np.zeros(n, np.int32)
        parent = np.zeros(n, np.int32)
        lcp = np.zeros(n + 1, np.int32)
        check(self._L.ncl_sparse_symbolic(self._h, ip(perm), ip(parent), ip(lcp)), "symbolic")
        return dict(perm=perm, parent=parent, lcol_ptr=lcp, l_nnz=int(lcp[-1]) if n else 0)

    def factorize(self, pivot_eps: float = 1e-10):
        info = np.zeros(4, np.int32)
        check(self._L.ncl_sparse_factorize(self._h, float(pivot_eps), ip(info)), "factorize")
        out = dict(ok=bool(info[0]), n_pos=int(info[1]), n_neg=int(info[2]), n_zero=0,
                   perturbed=int(info[3]))
        lcp = np.zeros(self.n + 1, np.int32)
        lri = np.zeros(self.l_nnz, np.int32)
        lv = np.zeros(self.l_nnz)
        d = np.zeros(self.n)
        check(self._L.ncl_sparse_factors(self._h, ip(lcp), ip(lri), dp(lv), dp(d)), "factors")
        out.update(lcol_ptr=lcp, lrow_ind=lri, lval=lv, d=d)
        return out

    def ldl_solve(self, b):
        b = f64(b)
        x = np.zeros(self.n)
        check(self._L.ncl_sparse_ldl_solve(self._h, dp(b), dp(x)), "ldl_solve")
        return x

    def solve_refined(self, b, max_ref: int = 10, tol: float = 1e-12):
        b = f64(b)
        x = np.zeros(self.n)
        steps = C.c_int()
        rel = C.c_double()
        conv = C.c_int()
        check(self._L.ncl_sparse_solve_refined(self._h, dp(b), int(max_ref), float(tol), dp(x),
                                               C.byref(steps), C.byref(rel), C.byref(conv)),
              "solve_refined")
        return x, steps.value, rel.value, bool(conv.value)


def analyze_host(n: int, rows, cols, perm=None):
    """analyze()/analyze_with_permutation() symbolic result, host only."""
    r, c = i32(rows), i32(cols)
    pm = None if perm is None else i32(perm)
    perm_o = np.zeros(n, np.int32)
    parent = np.zeros(n, np.int32)
    lcp = np.zeros(n + 1, np.int32)
    check(lib().ncl_analyze_host(n, len(r), ip(r), ip(c), ip(pm), ip(perm_o), ip(parent), ip(lcp)),
          "analyze")
    return dict(perm=perm_o, parent=parent, lcol_ptr=lcp, l_nnz=int(lcp[-1]) if n else 0)
