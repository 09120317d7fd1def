"""Shared test helpers: the reference tests' fixtures restated
(proj/tests/oracles.hpp, test_sparse.cpp:18-89, test_kkt.cpp:19-152)."""
import glob
import os

import numpy as np

from oracle import oracle as O
from paper_2510_05885_b200.instances import MT19937_64

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Rng:
    """oracles.hpp:109-119 (raw mt19937_64 bits)."""

    def __init__(self, seed):
        self.g = MT19937_64(seed)

    def uniform(self, lo=0.0, hi=1.0):
        return float(self.g.uniform(lo, hi, 1)[0])

    def uniform_int(self, lo, hi):
        return lo + int(int(self.g.raw(1)[0]) % (hi - lo + 1))


def from_dense_lower(M):
    """test_sparse.cpp:18-30: triplets of the nonzero lower triangle."""
    n = M.shape[0]
    ri, ci, v = [], [], []
    for j in range(n):
        for i in range(j, n):
            if M[i, j] != 0.0:
                ri.append(i)
                ci.append(j)
                v.append(M[i, j])
    return n, np.array(ri, np.int32), np.array(ci, np.int32), np.array(v)


def to_dense(n, col_ptr, row_ind, val):
    M = np.zeros((n, n))
    for j in range(n):
        for p in range(col_ptr[j], col_ptr[j + 1]):
            M[row_ind[p], j] = val[p]
            M[j, row_ind[p]] = val[p]
    return M


def random_sqd(n1, n2, seed):
    """test_sparse.cpp:55-87"""
    rng = Rng(seed)
    n = n1 + n2
    M = np.zeros((n, n))
    for b in range(2):
        lo, hi = (0, n1) if b == 0 else (n1, n)
        sgn = 1.0 if b == 0 else -1.0
        for j in range(lo, hi):
            for _ in range(3):
                i = rng.uniform_int(lo, hi - 1)
                if i != j:
                    v = rng.uniform(-1.0, 1.0)
                    M[max(i, j), min(i, j)] += sgn * v
        for j in range(lo, hi):
            rowsum = 0.0
            for i in range(lo, hi):
                if i != j:
                    rowsum += abs(M[max(i, j), min(i, j)])
            M[j, j] = sgn * (rowsum + 1.0 + rng.uniform(0.0, 1.0))
    for j in range(n1):
        for _ in range(2):
            i = rng.uniform_int(n1, n - 1)
            M[i, j] += rng.uniform(-1.0, 1.0)
    return M


def reconstruction_error(A_dense, perm, F):
    """test_sparse.cpp:32-47: max |P A P^T - L D L^T|"""
    n = A_dense.shape[0]
    P = np.zeros((n, n))
    P[np.arange(n), perm] = 1.0
    L = np.eye(n)
    lcp, lri, lv = F["lcol_ptr"], F["lrow_ind"], F["lval"]
    for j in range(n):
        for p in range(lcp[j], lcp[j + 1]):
            L[lri[p], j] = lv[p]
    return np.abs(P @ A_dense @ P.T - L @ np.diag(F["d"]) @ L.T).max()


def trivial_problem(nt, hdiag, rows, m_eq, jvals):
    """test_kkt.cpp:116-139 ("trivial_shape")"""
    hp_ptr = np.arange(nt + 1, dtype=np.int32)
    hp_idx = np.arange(nt, dtype=np.int32)
    jp_ptr = np.zeros(len(rows) + 1, np.int32)
    idx = []
    for i, r in enumerate(rows):
        jp_ptr[i + 1] = jp_ptr[i] + len(r)
        idx += list(r)
    m = len(rows)
    prob = O.Problem("trivial", nt, m - m_eq, m_eq, m, hp_ptr, hp_idx, jp_ptr,
                     np.array(idx, np.int32))
    return prob, np.array(hdiag, float), np.array(jvals, float)


def plain_case(prob, hval, jval, rho, rbar1, rbar2, rbar3):
    """test_kkt.cpp:141-152 ("plain_input"): sigma = 0"""
    return O.KktCase(hval, jval, np.zeros(prob.n), np.asarray(rbar1, float),
                     np.asarray(rbar2, float), np.asarray(rbar3, float), rho)


def golden_kkt_files():
    return sorted(glob.glob(os.path.join(GOLDEN, "kkt_*.npz")))


def load_golden(path):
    z = np.load(path, allow_pickle=False)
    prob = O.Problem(os.path.basename(path), int(z["nt"]), int(z["ns"]), int(z["m_eq"]), int(z["m"]),
                     z["hp_ptr"], z["hp_idx"], z["jp_ptr"], z["jp_idx"], z["lb"], z["ub"], z["start"])
    case = O.KktCase(z["hval"], z["jval"], z["sigma"], z["rbar1"], z["rbar2"], z["rbar3"], float(z["rho"]))
    return z, prob, case


def problem_from_instance(inst):
    return O.Problem(inst.name, inst.nt, inst.ns, inst.m_eq, inst.m, inst.hp_ptr, inst.hp_idx,
                     inst.jp_ptr, inst.jp_idx, inst.lb, inst.ub, inst.start)


def case_from_dict(d):
    return O.KktCase(d["hval"], d["jval"], d["sigma"], d["rbar1"], d["rbar2"], d["rbar3"], d["rho"])


def gpu_context(prob, form, opts=None):
    import paper_2510_05885_b200 as P
    hp = P.HessianPattern(prob.nt, prob.hp_ptr, prob.hp_idx)
    jp = P.JacobianPattern(prob.m, prob.nt, prob.jp_ptr, prob.jp_idx)
    o = None if opts is None else P.KktOptions(*opts)
    return P.KktContext(hp, jp, prob.nt, prob.ns, prob.m_eq, P.parse_kkt_form(form), o)


def gpu_input(case):
    import paper_2510_05885_b200 as P
    return P.KktInput(case.hval, case.jval, case.sigma, case.rbar1, case.rbar2, case.rbar3, case.rho)
