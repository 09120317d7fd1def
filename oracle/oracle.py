"""ctypes front for the oracle libraries -- TEST INFRASTRUCTURE ONLY.

Two libraries are wrapped:

* ``_ref/libncl_oracle.so``: the plain-C restatement (``ncl_oracle.c``), the
  parity checker.  Always buildable (gcc only).
* ``_ref/libncl_ref.so``: the reference's own sources (proj/src/*.cpp)
  compiled unmodified against ``eigen_shim`` plus ``ref_harness.cpp``.  Only
  buildable where /root/reference exists; prebuilt copies travel to the GPU
  box inside the snapshot.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBDIR = os.path.join(HERE, "_ref")

_i = C.c_int
_d = C.c_double
_p = C.c_void_p
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)

K2, K2R, K1S = 0, 1, 2
FORMS = {"k2": K2, "k2r": K2R, "k1s": K1S}


def _ip_(a):
    return a.ctypes.data_as(_ip) if a is not None else None


def _dp_(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def build(ref: bool = True) -> None:
    """Build the restatement (and the reference library when its sources are
    present in this container)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


_ORC = None
_REF = None


class OrcCsc(C.Structure):
    _fields_ = [("n", _i), ("nnz", _i), ("col_ptr", _ip), ("row_ind", _ip),
                ("val", _dp)]


class OrcSymbolic(C.Structure):
    _fields_ = [("n", _i), ("perm", _ip), ("iperm", _ip), ("parent", _ip),
                ("lcol_ptr", _ip), ("a_col_ptr", _ip), ("a_row_ind", _ip),
                ("a_map", _ip), ("nnz", _i)]


class OrcFactors(C.Structure):
    _fields_ = [("n", _i), ("ok", _i), ("lcol_ptr", _ip), ("lrow_ind", _ip),
                ("lval", _dp), ("d", _dp), ("n_pos", _i), ("n_neg", _i),
                ("n_zero", _i), ("perturbed", _i), ("pivot_eps", _d)]


class OrcKktOpts(C.Structure):
    _fields_ = [("pivot_eps", _d), ("max_refine", _i), ("refine_tol", _d),
                ("delta_max", _d), ("accept_tol", _d)]


class OrcKktStats(C.Structure):
    _fields_ = [("delta", _d), ("factor_attempts", _i), ("refine_steps", _i),
                ("perturbed_pivots", _i), ("rel_residual", _d), ("ok", _i)]


def orc():
    global _ORC
    if _ORC is None:
        path = os.path.join(LIBDIR, "libncl_oracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        L.orc_sym_from_triplets.argtypes = [_i, _i, _ip, _ip, _dp, C.POINTER(OrcCsc)]
        L.orc_csc_free.argtypes = [C.POINTER(OrcCsc)]
        L.orc_sym_matvec.argtypes = [C.POINTER(OrcCsc), _dp, _dp]
        L.orc_amd_order.argtypes = [C.POINTER(OrcCsc), _ip]
        L.orc_analyze_with_permutation.argtypes = [C.POINTER(OrcCsc), _ip, C.POINTER(OrcSymbolic)]
        L.orc_analyze.argtypes = [C.POINTER(OrcCsc), C.POINTER(OrcSymbolic)]
        L.orc_symbolic_free.argtypes = [C.POINTER(OrcSymbolic)]
        L.orc_factorize.argtypes = [C.POINTER(OrcSymbolic), C.POINTER(OrcCsc), _d, C.POINTER(OrcFactors)]
        L.orc_factors_free.argtypes = [C.POINTER(OrcFactors)]
        L.orc_ldl_solve.argtypes = [C.POINTER(OrcSymbolic), C.POINTER(OrcFactors), _dp, _dp]
        L.orc_solve_refined.argtypes = [C.POINTER(OrcSymbolic), C.POINTER(OrcFactors), C.POINTER(OrcCsc),
                                        _dp, _i, _d, _dp, _dp, _ip]
        L.orc_solve_refined.restype = _i
        L.orc_kkt_create.argtypes = [_i, _ip, _ip, _i, _ip, _ip, _i, _i, _i, C.POINTER(OrcKktOpts)]
        L.orc_kkt_create.restype = _p
        L.orc_kkt_destroy.argtypes = [_p]
        L.orc_kkt_system_size.argtypes = [_p]
        L.orc_kkt_nnz.argtypes = [_p]
        L.orc_kkt_num_pairs.argtypes = [_p]
        L.orc_kkt_inertia_target.argtypes = [_p, _ip]
        L.orc_kkt_matrix.argtypes = [_p, _ip, _ip, _dp]
        L.orc_kkt_symbolic.argtypes = [_p]
        L.orc_kkt_symbolic.restype = C.POINTER(OrcSymbolic)
        L.orc_kkt_last_factors.argtypes = [_p]
        L.orc_kkt_last_factors.restype = C.POINTER(OrcFactors)
        L.orc_kkt_refill.argtypes = [_p, _dp, _dp, _dp, _d, _d]
        L.orc_kkt_build_rhs.argtypes = [_p, _dp, _dp, _dp, _dp, _dp, _d, _d, _dp]
        L.orc_kkt_solve.argtypes = [_p, _dp, _dp, _dp, _dp, _dp, _dp, _d, _d, _dp, _dp, _dp,
                                    C.POINTER(OrcKktStats)]
        L.orc_recover_bound_duals.argtypes = [_i, _dp, _dp, _dp, _dp, _dp, _d, _dp, _dp, _dp]
        L.orc_barrier_kkt_residual.argtypes = [_i, _i, _i, _ip, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _d,
                                               _dp, _dp, _dp, _dp, _dp, _d, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_fraction_to_boundary.argtypes = [_i, _dp, _dp, _dp, _dp, _d]
        L.orc_fraction_to_boundary.restype = _d
        L.orc_dual_fraction_to_boundary.argtypes = [_i, _dp, _dp, _d]
        L.orc_dual_fraction_to_boundary.restype = _d
        L.orc_clip_duals.argtypes = [_i, _dp, _dp, _dp, _d, _dp, _dp]
        L.orc_kkt_input.argtypes = [_i, _i, _i, _ip, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                    _dp, _dp, _d, _d, _dp, _dp, _dp, _dp]
        L.orc_initial_outer_state.argtypes = [_d, _d, _d, _dp]
        L.orc_outer_update.argtypes = [_dp, _d]
        L.orc_outer_update.restype = _i
        L.orc_init_multipliers.argtypes = [_i, _i, _ip, _ip, _dp, _dp, _dp]
        _ORC = L
    return _ORC


def ref_available() -> bool:
    return os.path.exists(os.path.join(LIBDIR, "libncl_ref.so"))


def ref():
    global _REF
    if _REF is None:
        path = os.path.join(LIBDIR, "libncl_ref.so")
        if not os.path.exists(path):
            build(ref=True)
        L = C.CDLL(path)
        L.ref_model_new.argtypes = [C.c_char_p]
        L.ref_model_new.restype = _p
        L.ref_model_free.argtypes = [_p]
        L.ref_model_dims.argtypes = [_p, _ip]
        L.ref_model_patterns.argtypes = [_p, _ip, _ip, _ip, _ip]
        L.ref_model_bounds.argtypes = [_p, _dp, _dp, _dp]
        L.ref_model_eval.argtypes = [_p, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_kkt_case.argtypes = [_p, C.c_uint, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_kkt_new.argtypes = [_i, _ip, _ip, _i, _ip, _ip, _i, _i, _i, _dp]
        L.ref_kkt_new.restype = _p
        L.ref_kkt_free.argtypes = [_p]
        L.ref_kkt_size.argtypes = [_p]
        L.ref_kkt_nnz.argtypes = [_p]
        L.ref_kkt_matrix.argtypes = [_p, _ip, _ip, _dp]
        L.ref_kkt_solve_n.argtypes = [_p, _i, _dp, _dp, _dp, _dp, _dp, _dp, _d, _d, _dp, _dp, _dp, _dp]
        L.ref_sparse_new.argtypes = [_i, _i, _ip, _ip, _dp, _ip]
        L.ref_sparse_new.restype = _p
        L.ref_sparse_free.argtypes = [_p]
        L.ref_sparse_nnz.argtypes = [_p]
        L.ref_sparse_lnz.argtypes = [_p]
        L.ref_sparse_matrix.argtypes = [_p, _ip, _ip, _dp]
        L.ref_sparse_symbolic.argtypes = [_p, _ip, _ip, _ip, _ip]
        L.ref_sparse_factorize.argtypes = [_p, _d, _ip, _ip, _dp, _dp]
        L.ref_sparse_solve_refined.argtypes = [_p, _dp, _i, _d, _dp, _dp]
        L.ref_sparse_solve_refined.restype = _i
        L.ref_sparse_ldl_solve.argtypes = [_p, _dp, _dp]
        L.ref_solve.argtypes = [_p, _i, _d, _i, _i, _d, _i]
        L.ref_solve.restype = _p
        L.ref_report_free.argtypes = [_p]
        L.ref_report_scalars.argtypes = [_p, _dp]
        L.ref_report_log.argtypes = [_p, _dp, _dp]
        L.ref_report_xy.argtypes = [_p, _dp, _dp]
        L.ref_time_init_multipliers.argtypes = [_p]
        L.ref_time_init_multipliers.restype = _d
        _REF = L
    return _REF


# ---------------------------------------------------------------- data types
@dataclass
class Problem:
    """Patterns of one NLP in the reference's conventions (model.hpp:38-48)."""
    name: str
    nt: int
    ns: int
    m_eq: int
    m: int
    hp_ptr: np.ndarray
    hp_idx: np.ndarray
    jp_ptr: np.ndarray
    jp_idx: np.ndarray
    lb: np.ndarray = None
    ub: np.ndarray = None
    start: np.ndarray = None

    @property
    def n(self):
        return self.nt + self.ns


@dataclass
class KktCase:
    hval: np.ndarray
    jval: np.ndarray
    sigma: np.ndarray
    rbar1: np.ndarray
    rbar2: np.ndarray
    rbar3: np.ndarray
    rho: float = 100.0


@dataclass
class Step:
    dx: np.ndarray
    dr: np.ndarray
    dy: np.ndarray
    delta: float
    factor_attempts: int
    refine_steps: int
    perturbed_pivots: int
    rel_residual: float
    ok: bool


# ------------------------------------------------------- reference model API
class RefModel:
    """A reference ``ncl::Model`` built from an instance spec (see
    integration/instances.hpp)."""

    def __init__(self, spec: str):
        L = ref()
        self.L = L
        self.h = L.ref_model_new(spec.encode())
        if not self.h:
            raise ValueError(f"unknown instance {spec}")
        d = np.zeros(6, np.int32)
        L.ref_model_dims(self.h, _ip_(d))
        self.nt, self.ns, self.m_eq, self.m, self.hnnz, self.jnnz = map(int, d)
        self.n = self.nt + self.ns
        hp_ptr = np.zeros(self.nt + 1, np.int32)
        hp_idx = np.zeros(self.hnnz, np.int32)
        jp_ptr = np.zeros(self.m + 1, np.int32)
        jp_idx = np.zeros(self.jnnz, np.int32)
        L.ref_model_patterns(self.h, _ip_(hp_ptr), _ip_(hp_idx), _ip_(jp_ptr), _ip_(jp_idx))
        lb = np.zeros(self.n)
        ub = np.zeros(self.n)
        st = np.zeros(self.nt)
        L.ref_model_bounds(self.h, _dp_(lb), _dp_(ub), _dp_(st))
        self.problem = Problem(spec, self.nt, self.ns, self.m_eq, self.m, hp_ptr, hp_idx,
                               jp_ptr, jp_idx, lb, ub, st)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_model_free(self.h)
            self.h = None

    def kkt_case(self, seed: int, rho: float = 100.0) -> KktCase:
        hv = np.zeros(self.hnnz)
        jv = np.zeros(self.jnnz)
        sg = np.zeros(self.n)
        r1 = np.zeros(self.n)
        r2 = np.zeros(self.m)
        r3 = np.zeros(self.m)
        self.L.ref_kkt_case(self.h, seed, _dp_(hv), _dp_(jv), _dp_(sg), _dp_(r1), _dp_(r2), _dp_(r3))
        return KktCase(hv, jv, sg, r1, r2, r3, rho)

    def eval(self, t, y):
        hv = np.zeros(self.hnnz)
        jv = np.zeros(self.jnnz)
        g = np.zeros(self.nt)
        c = np.zeros(self.m)
        self.L.ref_model_eval(self.h, _dp_(f64(t)), _dp_(f64(y)), _dp_(hv), _dp_(jv), _dp_(g), _dp_(c))
        return hv, jv, g, c

    def solve(self, form="k1s", tol=1e-8, max_outer=40, max_inner=1000, pivot_eps=1e-10, scaling=True):
        L = self.L
        r = L.ref_solve(self.h, FORMS[form], tol, max_outer, max_inner, pivot_eps, int(scaling))
        sc = np.zeros(12)
        L.ref_report_scalars(r, _dp_(sc))
        nlog, nex = int(sc[10]), int(sc[11])
        log = np.zeros((max(nlog, 1), 13))
        ex = np.zeros(max(nex, 1))
        L.ref_report_log(r, _dp_(log), _dp_(ex))
        x = np.zeros(self.n)
        y = np.zeros(self.m)
        L.ref_report_xy(r, _dp_(x), _dp_(y))
        L.ref_report_free(r)
        status = ["optimal", "infeasible", "iteration_limit", "numeric_error"][int(sc[0])]
        return dict(status=status, outer_iters=int(sc[1]), inner_iters=int(sc[2]),
                    extrapolation_accepts=int(sc[3]), objective=sc[4], kkt_residual=sc[5],
                    primal_feas=sc[6], mu_final=sc[7], rho_final=sc[8], solve_seconds=sc[9],
                    log=log[:nlog], extrap_alpha=ex[:nex], x=x, y=y)


class RefKkt:
    """The reference's own ``ncl::KktContext`` (proj/src/kkt.cpp)."""

    def __init__(self, prob: Problem, form: str, opts=None):
        L = ref()
        self.L = L
        self.prob = prob
        o = None if opts is None else f64(opts)
        self.h = L.ref_kkt_new(prob.nt, _ip_(i32(prob.hp_ptr)), _ip_(i32(prob.hp_idx)), prob.m,
                               _ip_(i32(prob.jp_ptr)), _ip_(i32(prob.jp_idx)), prob.ns, prob.m_eq,
                               FORMS[form], _dp_(o))
        if not self.h:
            raise ValueError("kkt: invalid shape")
        self.N = L.ref_kkt_size(self.h)
        self.nnz = L.ref_kkt_nnz(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_kkt_free(self.h)
            self.h = None

    def solve(self, c: KktCase, warm_delta=0.0) -> Step:
        p = self.prob
        dx = np.zeros(p.n)
        dr = np.zeros(p.m)
        dy = np.zeros(p.m)
        st = np.zeros(6)
        self.L.ref_kkt_solve_n(self.h, p.n, _dp_(f64(c.hval)), _dp_(f64(c.jval)), _dp_(f64(c.sigma)),
                               _dp_(f64(c.rbar1)), _dp_(f64(c.rbar2)), _dp_(f64(c.rbar3)), c.rho,
                               warm_delta, _dp_(dx), _dp_(dr), _dp_(dy), _dp_(st))
        return Step(dx, dr, dy, st[0], int(st[1]), int(st[2]), int(st[3]), st[4], bool(st[5]))

    def matrix(self):
        cp = np.zeros(self.N + 1, np.int32)
        ri = np.zeros(self.nnz, np.int32)
        v = np.zeros(self.nnz)
        self.L.ref_kkt_matrix(self.h, _ip_(cp), _ip_(ri), _dp_(v))
        return cp, ri, v


# ------------------------------------------------------------ restatement API
class OrcKkt:
    """The C restatement of ``ncl::KktContext`` (oracle/ncl_oracle.c)."""

    def __init__(self, prob: Problem, form: str, opts=None):
        L = orc()
        self.L = L
        self.prob = prob
        o = None
        if opts is not None:
            o = OrcKktOpts(*opts)
        self._keep = [i32(prob.hp_ptr), i32(prob.hp_idx), i32(prob.jp_ptr), i32(prob.jp_idx)]
        self.h = L.orc_kkt_create(prob.nt, _ip_(self._keep[0]), _ip_(self._keep[1]), prob.m,
                                  _ip_(self._keep[2]), _ip_(self._keep[3]), prob.ns, prob.m_eq,
                                  FORMS[form], C.byref(o) if o is not None else None)
        if not self.h:
            raise ValueError("kkt: inconsistent problem shape")
        self.N = L.orc_kkt_system_size(self.h)
        self.nnz = L.orc_kkt_nnz(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_kkt_destroy(self.h)
            self.h = None

    def inertia_target(self):
        t = np.zeros(3, np.int32)
        self.L.orc_kkt_inertia_target(self.h, _ip_(t))
        return tuple(int(v) for v in t)

    def solve(self, c: KktCase, warm_delta=0.0) -> Step:
        p = self.prob
        dx = np.zeros(p.n)
        dr = np.zeros(p.m)
        dy = np.zeros(p.m)
        st = OrcKktStats()
        self.L.orc_kkt_solve(self.h, _dp_(f64(c.hval)), _dp_(f64(c.jval)), _dp_(f64(c.sigma)),
                             _dp_(f64(c.rbar1)), _dp_(f64(c.rbar2)), _dp_(f64(c.rbar3)), c.rho,
                             warm_delta, _dp_(dx), _dp_(dr), _dp_(dy), C.byref(st))
        return Step(dx, dr, dy, st.delta, st.factor_attempts, st.refine_steps, st.perturbed_pivots,
                    st.rel_residual, bool(st.ok))

    def refill(self, c: KktCase, delta=0.0):
        self.L.orc_kkt_refill(self.h, _dp_(f64(c.hval)), _dp_(f64(c.jval)), _dp_(f64(c.sigma)), c.rho, delta)
        return self.matrix()[2]

    def build_rhs(self, c: KktCase, delta=0.0):
        rhs = np.zeros(self.N)
        self.L.orc_kkt_build_rhs(self.h, _dp_(f64(c.jval)), _dp_(f64(c.sigma)), _dp_(f64(c.rbar1)),
                                 _dp_(f64(c.rbar2)), _dp_(f64(c.rbar3)), c.rho, delta, _dp_(rhs))
        return rhs

    def matrix(self):
        cp = np.zeros(self.N + 1, np.int32)
        ri = np.zeros(self.nnz, np.int32)
        v = np.zeros(self.nnz)
        self.L.orc_kkt_matrix(self.h, _ip_(cp), _ip_(ri), _dp_(v))
        return cp, ri, v

    def symbolic(self):
        S = self.L.orc_kkt_symbolic(self.h).contents
        n = S.n
        g = lambda ptr, k: np.ctypeslib.as_array(ptr, shape=(k,)).copy() if k else np.zeros(0, np.int32)
        return dict(perm=g(S.perm, n), iperm=g(S.iperm, n), parent=g(S.parent, n),
                    lcol_ptr=g(S.lcol_ptr, n + 1), a_col_ptr=g(S.a_col_ptr, n + 1),
                    a_row_ind=g(S.a_row_ind, S.nnz), a_map=g(S.a_map, S.nnz))

    def last_factors(self):
        P = self.L.orc_kkt_last_factors(self.h)
        if not P:
            return None
        F = P.contents
        n = F.n
        lnz = F.lcol_ptr[n]
        g = lambda ptr, k, dt: np.ctypeslib.as_array(ptr, shape=(k,)).copy() if k else np.zeros(0, dt)
        return dict(ok=bool(F.ok), n_pos=F.n_pos, n_neg=F.n_neg, perturbed=F.perturbed,
                    lcol_ptr=g(F.lcol_ptr, n + 1, np.int32), lrow_ind=g(F.lrow_ind, lnz, np.int32),
                    lval=g(F.lval, lnz, np.float64), d=g(F.d, n, np.float64))


class OrcSparse:
    """sparse.cpp restated: triplets -> analyze -> factorize -> solves."""

    def __init__(self, n, rows, cols, vals, perm=None):
        L = orc()
        self.L = L
        self.A = OrcCsc()
        rows, cols, vals = i32(rows), i32(cols), f64(vals)
        if L.orc_sym_from_triplets(n, len(rows), _ip_(rows), _ip_(cols), _dp_(vals), C.byref(self.A)):
            raise ValueError("sym_from_triplets: index out of range")
        self.S = OrcSymbolic()
        if perm is None:
            rc = L.orc_analyze(C.byref(self.A), C.byref(self.S))
        else:
            pm = i32(perm)
            rc = L.orc_analyze_with_permutation(C.byref(self.A), _ip_(pm), C.byref(self.S))
        if rc:
            raise ValueError("analyze: invalid input")
        self.F = None
        self.n = n

    def __del__(self):
        if getattr(self, "L", None) is None:
            return
        if self.F is not None:
            self.L.orc_factors_free(C.byref(self.F))
        self.L.orc_symbolic_free(C.byref(self.S))
        self.L.orc_csc_free(C.byref(self.A))

    def matrix(self):
        n, nz = self.A.n, self.A.nnz
        return (np.ctypeslib.as_array(self.A.col_ptr, shape=(n + 1,)).copy(),
                np.ctypeslib.as_array(self.A.row_ind, shape=(nz,)).copy() if nz else np.zeros(0, np.int32),
                np.ctypeslib.as_array(self.A.val, shape=(nz,)).copy() if nz else np.zeros(0))

    def symbolic(self):
        S = self.S
        n = S.n
        g = lambda ptr, k: np.ctypeslib.as_array(ptr, shape=(k,)).copy() if k else np.zeros(0, np.int32)
        return dict(perm=g(S.perm, n), parent=g(S.parent, n), lcol_ptr=g(S.lcol_ptr, n + 1),
                    a_map=g(S.a_map, S.nnz), l_nnz=int(S.lcol_ptr[n]) if n else 0)

    def factorize(self, eps=1e-10):
        if self.F is not None:
            self.L.orc_factors_free(C.byref(self.F))
        self.F = OrcFactors()
        self.L.orc_factorize(C.byref(self.S), C.byref(self.A), eps, C.byref(self.F))
        F = self.F
        n = F.n
        lnz = F.lcol_ptr[n] if n else 0
        g = lambda ptr, k, dt: np.ctypeslib.as_array(ptr, shape=(k,)).copy() if k else np.zeros(0, dt)
        return dict(ok=bool(F.ok), n_pos=F.n_pos, n_neg=F.n_neg, n_zero=F.n_zero, perturbed=F.perturbed,
                    lcol_ptr=g(F.lcol_ptr, n + 1, np.int32), lrow_ind=g(F.lrow_ind, lnz, np.int32),
                    lval=g(F.lval, lnz, np.float64), d=g(F.d, n, np.float64))

    def ldl_solve(self, b):
        x = np.zeros(self.n)
        self.L.orc_ldl_solve(C.byref(self.S), C.byref(self.F), _dp_(f64(b)), _dp_(x))
        return x

    def solve_refined(self, b, max_ref=10, tol=1e-12):
        x = np.zeros(self.n)
        rel = C.c_double()
        conv = C.c_int()
        steps = self.L.orc_solve_refined(C.byref(self.S), C.byref(self.F), C.byref(self.A), _dp_(f64(b)),
                                         max_ref, tol, _dp_(x), C.byref(rel), C.byref(conv))
        return x, steps, rel.value, bool(conv.value)

    def matvec(self, x, y=None):
        y = np.zeros(self.n) if y is None else f64(y).copy()
        self.L.orc_sym_matvec(C.byref(self.A), _dp_(f64(x)), _dp_(y))
        return y
