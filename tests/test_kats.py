"""Known-answer tests of the reference (proj/tests/test_sparse.cpp,
test_kkt.cpp, test_ipm.cpp, test_solver.cpp) restated, run against both the
CPU oracle (always) and the sm_100a path (marked gpu)."""
import ctypes as C

import numpy as np
import pytest

from helpers import (Rng, from_dense_lower, golden_kkt_files, load_golden, plain_case,
                     random_sqd, reconstruction_error, to_dense, trivial_problem)
from oracle import oracle as O

ENGINES = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


# ------------------------------------------------------------------ engines
def sparse_engine(kind, n, rows, cols, vals, perm=None):
    if kind == "oracle":
        return O.OrcSparse(n, rows, cols, vals, perm)
    import paper_2510_05885_b200 as P
    return P.SparseLdl(n, rows, cols, vals, perm)


class GpuKkt:
    def __init__(self, prob, form, opts=None):
        from helpers import gpu_context
        self.ctx = gpu_context(prob, form, opts)
        self.N = self.ctx.system_size()

    def solve(self, case, warm=0.0):
        from helpers import gpu_input
        return self.ctx.solve(gpu_input(case), warm)

    def matrix(self):
        return self.ctx.matrix()

    def inertia_target(self):
        return self.ctx.inertia_target()


def kkt_engine(kind, prob, form, opts=None):
    if kind == "oracle":
        return O.OrcKkt(prob, form, opts)
    return GpuKkt(prob, form, opts)


@pytest.fixture(params=ENGINES)
def engine(request):
    return request.param


# ------------------------------------------------------------- sparse KATs
def test_triplet_assembly_mirrors_and_sums_duplicates():
    """test_sparse.cpp:93-110"""
    S = O.OrcSparse(2, [0, 0, 1, 1], [0, 1, 1, 1], [2.0, 1.0, -1.0, -2.0])
    cp, ri, v = S.matrix()
    assert cp[-1] == 3
    D = to_dense(2, cp, ri, v)
    assert D[0, 0] == 2.0 and D[1, 0] == 1.0 and D[0, 1] == 1.0 and D[1, 1] == -3.0
    for j in range(2):
        for p in range(cp[j], cp[j + 1]):
            assert ri[p] >= j
            if p > cp[j]:
                assert ri[p] > ri[p - 1]


def test_diagonal_pattern_has_zero_fill(engine):
    """test_sparse.cpp:112-120"""
    n = 7
    S = sparse_engine(engine, n, np.arange(n), np.arange(n), np.ones(n))
    assert S.symbolic()["l_nnz"] == 0


def test_amd_sends_arrowhead_hub_last(engine):
    """test_sparse.cpp:122-146"""
    n = 30
    ri = list(range(n)) + list(range(1, n))
    ci = list(range(n)) + [0] * (n - 1)
    v = [4.0] * n + [1.0] * (n - 1)
    nat = sparse_engine(engine, n, ri, ci, v, perm=np.arange(n))
    assert nat.symbolic()["l_nnz"] == n * (n - 1) // 2
    amd = sparse_engine(engine, n, ri, ci, v)
    sym = amd.symbolic()
    assert sym["l_nnz"] == n - 1
    assert sym["perm"][-1] == 0


def test_hand_computed_2x2_indefinite(engine):
    """test_sparse.cpp:148-163"""
    S = sparse_engine(engine, 2, [0, 1, 1], [0, 0, 1], [2.0, 1.0, -3.0], perm=[0, 1])
    F = S.factorize(1e-10)
    assert F["ok"]
    assert abs(F["d"][0] - 2.0) <= 1e-15 * 2.0
    assert abs(F["d"][1] + 3.5) <= 1e-15 * 3.5
    assert F["lcol_ptr"][1] - F["lcol_ptr"][0] == 1
    assert abs(F["lval"][0] - 0.5) <= 1e-15
    assert (F["n_pos"], F["n_neg"], F["perturbed"]) == (1, 1, 0)


def test_zero_matrix_perturbs_every_pivot(engine):
    """test_sparse.cpp:165-174"""
    S = sparse_engine(engine, 2, [0, 1], [0, 1], [0.0, 0.0])
    F = S.factorize(1e-10)
    assert F["ok"]
    assert F["d"][0] == 1e-10 and F["d"][1] == 1e-10
    assert F["perturbed"] == 2 and F["n_pos"] == 2


def test_pivot_eps_zero_aborts_on_exact_zero(engine):
    """test_sparse.cpp:176-181"""
    S = sparse_engine(engine, 2, [0, 1], [0, 1], [0.0, 1.0], perm=[0, 1])
    assert not S.factorize(0.0)["ok"]


def test_sqd_reconstructs_without_perturbation(engine):
    """test_sparse.cpp:183-193"""
    M = random_sqd(30, 20, 20240817)
    n, ri, ci, v = from_dense_lower(M)
    S = sparse_engine(engine, n, ri, ci, v)
    F = S.factorize(1e-10)
    assert F["ok"] and F["perturbed"] == 0
    assert (F["n_pos"], F["n_neg"]) == (30, 20)
    Md = np.tril(M) + np.tril(M, -1).T
    assert reconstruction_error(Md, S.symbolic()["perm"], F) <= 1e-12 * np.abs(Md).max()


def test_inertia_matches_dense_eigenvalues(engine):
    """test_sparse.cpp:195-220"""
    checked = 0
    for seed in (11, 22, 33, 44, 55, 66):
        rng = Rng(seed)
        n = rng.uniform_int(5, 60)
        M = np.zeros((n, n))
        for i in range(n):
            for j in range(i + 1):
                M[i, j] = rng.uniform(-1.0, 1.0)
                M[j, i] = M[i, j]
        M[np.diag_indices(n)] += rng.uniform(-2.0, 2.0)
        lam = np.linalg.eigvalsh(M)
        if np.any(np.abs(lam) <= 1e-8) or np.abs(lam).min() < 1e-6:
            continue
        n_, ri, ci, v = from_dense_lower(M)
        F = sparse_engine(engine, n_, ri, ci, v).factorize(1e-10)
        assert F["ok"]
        assert F["n_pos"] == int((lam > 1e-8).sum())
        assert F["n_neg"] == int((lam < -1e-8).sum())
        checked += 1
    assert checked >= 3


def test_random_sparse_reconstruction(engine):
    """test_sparse.cpp:222-241"""
    rng = Rng(777)
    n = 40
    M = np.zeros((n, n))
    for j in range(n):
        M[j, j] = rng.uniform(0.5, 3.0) * (-1.0 if rng.uniform() < 0.3 else 1.0)
        for _ in range(2):
            i = rng.uniform_int(0, n - 1)
            if i != j:
                M[max(i, j), min(i, j)] += rng.uniform(-0.3, 0.3)
    Ml = np.tril(M)
    Md = Ml + np.tril(Ml, -1).T
    n_, ri, ci, v = from_dense_lower(Ml)
    S = sparse_engine(engine, n_, ri, ci, v)
    F = S.factorize(1e-10)
    assert F["ok"]
    if F["perturbed"] == 0:
        assert reconstruction_error(Md, S.symbolic()["perm"], F) <= 1e-11 * np.abs(Md).max()


def test_factorization_bitwise_deterministic(engine):
    """test_sparse.cpp:243-252"""
    M = random_sqd(25, 15, 99)
    n, ri, ci, v = from_dense_lower(M)
    S1 = sparse_engine(engine, n, ri, ci, v)
    S2 = sparse_engine(engine, n, ri, ci, v)
    assert np.array_equal(S1.symbolic()["perm"], S2.symbolic()["perm"])
    F1, F2 = S1.factorize(1e-10), S2.factorize(1e-10)
    assert np.array_equal(F1["lval"].view(np.int64), F2["lval"].view(np.int64))
    assert np.array_equal(F1["d"].view(np.int64), F2["d"].view(np.int64))


def test_identity_needs_zero_refinements(engine):
    """test_sparse.cpp:254-265"""
    S = sparse_engine(engine, 3, [0, 1, 2], [0, 1, 2], [1.0, 1.0, 1.0])
    S.factorize(1e-10)
    x, steps, rel, conv = S.solve_refined(np.array([1.0, -2.0, 3.0]))
    assert conv and steps == 0
    assert list(x) == [1.0, -2.0, 3.0]


def test_refinement_recovers_through_perturbed_pivot(engine):
    """test_sparse.cpp:267-281"""
    S = sparse_engine(engine, 2, [0, 1], [0, 1], [1.0, 9e-11], perm=[0, 1])
    F = S.factorize(1e-10)
    assert F["ok"] and F["perturbed"] == 1
    x, steps, rel, conv = S.solve_refined(np.array([1.0, 9e-11]), 10, 1e-20)
    assert abs(x[0] - 1.0) <= 1e-12
    assert abs(x[1] - 1.0) <= 1e-8
    assert steps <= 10


def test_kappa_1e14_is_residual_converged_only(engine):
    """test_sparse.cpp:283-298"""
    S = sparse_engine(engine, 2, [0, 1], [0, 1], [1.0, 1e-14], perm=[0, 1])
    F = S.factorize(1e-10)
    assert F["ok"] and F["perturbed"] == 1
    x, steps, rel, conv = S.solve_refined(np.array([1.0, 1e-14]))
    assert conv and rel <= 1e-12
    assert abs(x[1] - 1e-4) <= 1e-6


def test_refinement_never_worse(engine):
    """test_sparse.cpp:300-322"""
    M = random_sqd(20, 12, 4242)
    n, ri, ci, v = from_dense_lower(M)
    S = sparse_engine(engine, n, ri, ci, v)
    assert S.factorize(1e-10)["ok"]
    rng = Rng(5)
    b = np.array([rng.uniform(-1.0, 1.0) for _ in range(n)])
    x0 = S.ldl_solve(b)
    Md = np.tril(M) + np.tril(M, -1).T
    plain = np.abs(Md @ x0 - b).max()
    x, steps, rel, conv = S.solve_refined(b)
    assert rel * np.abs(b).max() <= plain * (1.0 + 1e-15)


# --------------------------------------------------------------- KKT KATs
def golden(name):
    for p in golden_kkt_files():
        if p.endswith(f"kkt_{name}.npz"):
            return load_golden(p)
    raise FileNotFoundError(name)


def dense_blocks(prob, hval, jval):
    n = prob.n
    W = np.zeros((n, n))
    for j in range(prob.nt):
        for p in range(prob.hp_ptr[j], prob.hp_ptr[j + 1]):
            W[prob.hp_idx[p], j] = hval[p]
            W[j, prob.hp_idx[p]] = hval[p]
    J = np.zeros((prob.m, n))
    for i in range(prob.m):
        for p in range(prob.jp_ptr[i], prob.jp_ptr[i + 1]):
            J[i, prob.jp_idx[p]] = jval[p]
    for k in range(prob.ns):
        J[prob.m_eq + k, prob.nt + k] = -1.0
    return W, J


def newton_residual(prob, case, st):
    """test_kkt.cpp:91-107"""
    W, J = dense_blocks(prob, case.hval, case.jval)
    rho_hat = case.rho + st.delta
    e1 = W @ st.dx - J.T @ st.dy + case.rbar1 + (case.sigma + st.delta) * st.dx
    e2 = rho_hat * st.dr - st.dy + case.rbar2
    e3 = J @ st.dx + st.dr + case.rbar3
    r = np.abs(e1).max()
    if len(e2):
        r = max(r, np.abs(e2).max(), np.abs(e3).max())
    return r


def step_scale(st):
    s = max(1.0, np.abs(st.dx).max())
    return max(s, np.abs(st.dy).max()) if len(st.dy) else s


def test_inertia_targets_per_form(engine):
    """test_kkt.cpp:166-181"""
    _, prob, _ = golden("hs35")
    sizes = {}
    for form, tgt in (("k2", (5, 1, 0)), ("k2r", (4, 1, 0)), ("k1s", (3, 0, 0))):
        K = kkt_engine(engine, prob, form)
        sizes[form] = K.N
        assert tuple(K.inertia_target()) == tgt
    assert sizes == {"k2": 6, "k2r": 5, "k1s": 3}


def test_two_by_two_reduced_system_solves_exactly(engine):
    """test_kkt.cpp:183-197"""
    prob, hv, jv = trivial_problem(1, [2.0], [[0]], 1, [1.0])
    case = plain_case(prob, hv, jv, 1.0, [-1.0], [0.0], [-1.0])
    for form in ("k2", "k2r", "k1s"):
        st = kkt_engine(engine, prob, form).solve(case, 0.0)
        assert st.ok and st.delta == 0.0
        assert abs(st.dx[0] - 2.0 / 3.0) <= 1e-12 * 2.0 / 3.0
        assert abs(st.dy[0] - 1.0 / 3.0) <= 1e-12 / 3.0
        assert abs(st.dr[0] - 1.0 / 3.0) <= 1e-12 / 3.0


@pytest.mark.parametrize("name", ["hs35", "redundant_circle", "opf_toy_30"])
def test_three_forms_agree(engine, name):
    """test_kkt.cpp:199-221"""
    _, prob, case = golden(name)
    ref = None
    for form in ("k2", "k2r", "k1s"):
        st = kkt_engine(engine, prob, form).solve(case, 0.0)
        assert st.ok and st.delta == 0.0
        scale = step_scale(st)
        assert newton_residual(prob, case, st) <= 1e-7 * scale
        if ref is None:
            ref = st
        else:
            for k in ("dx", "dy", "dr"):
                assert np.abs(getattr(st, k) - getattr(ref, k)).max() <= 1e-7 * scale


def test_rank_deficient_jacobian_without_regularization(engine):
    """test_kkt.cpp:223-234 (dup-rows, seed 7)"""
    M = None
    try:
        M = O.RefModel("dup-rows")
    except Exception:
        pass
    if M is None:
        pytest.skip("reference library not built here")
    prob, case = M.problem, M.kkt_case(7)
    for form in ("k2", "k2r", "k1s"):
        st = kkt_engine(engine, prob, form).solve(case, 0.0)
        assert st.ok and st.delta == 0.0
        assert newton_residual(prob, case, st) <= 1e-7 * step_scale(st)


@pytest.mark.parametrize("sig_s,expect", [(1e8, 1.0 + 100.0 * (1e8 / (1e8 + 100.0))), (0.0, 1.0)])
def test_condensed_slack_weight(engine, sig_s, expect):
    """test_kkt.cpp:236-260"""
    prob, hv, jv = trivial_problem(1, [0.0], [[0]], 0, [1.0])
    case = plain_case(prob, hv, jv, 100.0, [0.0, 0.0], [0.0], [-1.0])
    case.sigma = np.array([1.0, sig_s])
    K = kkt_engine(engine, prob, "k1s")
    st = K.solve(case, 0.0)
    assert st.ok
    assert abs(K.matrix()[2][0] - expect) <= 1e-14 * expect


def test_zero_matrix_escalates_to_delta(engine):
    """test_kkt.cpp:262-274"""
    prob, hv, jv = trivial_problem(2, [0.0, 0.0], [], 0, [])
    case = plain_case(prob, hv, jv, 100.0, [-1.0, -1.0], [], [])
    st = kkt_engine(engine, prob, "k1s").solve(case, 0.0)
    assert st.ok and st.factor_attempts == 2
    assert abs(st.delta - 1e-8) <= 1e-14 * 1e-8
    assert np.all(np.abs(st.dx - 1e8) <= 1e-9 * 1e8)


def test_warm_delta_seeds_at_a_third(engine):
    """test_kkt.cpp:276-284"""
    prob, hv, jv = trivial_problem(2, [0.0, 0.0], [], 0, [])
    case = plain_case(prob, hv, jv, 100.0, [-1.0, -1.0], [], [])
    st = kkt_engine(engine, prob, "k1s").solve(case, 9e-9)
    assert st.ok and st.factor_attempts == 2
    assert abs(st.delta - 3e-9) <= 1e-14 * 3e-9


def test_negative_curvature_frozen_escalation(engine):
    """test_kkt.cpp:286-298"""
    prob, hv, jv = trivial_problem(2, [-2.0, -2.0], [], 0, [])
    case = plain_case(prob, hv, jv, 100.0, [1.0, 1.0], [], [])
    for form in ("k2", "k2r", "k1s"):
        st = kkt_engine(engine, prob, form).solve(case, 0.0)
        assert st.ok and st.factor_attempts == 11
        want = 2e-8 * 8.0 ** 9
        assert abs(st.delta - want) <= 1e-13 * want
        assert abs(st.dx[0] - (-1.0 / (st.delta - 2.0))) <= 1e-10 * abs(1.0 / (st.delta - 2.0))


def test_cross_form_agreement_with_delta(engine):
    """test_kkt.cpp:300-322"""
    prob, hv, jv = trivial_problem(2, [-2.0, -2.0], [[0]], 1, [1.0])
    case = plain_case(prob, hv, jv, 100.0, [1.0, 1.0], [0.5], [-0.3])
    ref = None
    for form in ("k2", "k2r", "k1s"):
        st = kkt_engine(engine, prob, form).solve(case, 0.0)
        assert st.ok and st.delta > 0.0
        if ref is None:
            ref = st
        else:
            assert st.delta == ref.delta
            sc = step_scale(ref)
            for k in ("dx", "dy", "dr"):
                assert np.abs(getattr(st, k) - getattr(ref, k)).max() <= 1e-9 * sc


def test_exhausting_delta_reports_failure(engine):
    """test_kkt.cpp:324-333"""
    prob, hv, jv = trivial_problem(2, [-2.0, -2.0], [], 0, [])
    case = plain_case(prob, hv, jv, 100.0, [1.0, 1.0], [], [])
    st = kkt_engine(engine, prob, "k1s", opts=(1e-10, 10, 1e-12, 1e-7, 1e-8)).solve(case, 0.0)
    assert not st.ok and st.factor_attempts == 2


def test_inconsistent_shape_raises(engine):
    """kkt.cpp:52-53: ns must equal the inequality row count"""
    prob, hv, jv = trivial_problem(1, [1.0], [[0]], 1, [1.0])
    bad = O.Problem("bad", prob.nt, 1, prob.m_eq, prob.m, prob.hp_ptr, prob.hp_idx, prob.jp_ptr,
                    prob.jp_idx)
    with pytest.raises(ValueError):
        kkt_engine(engine, bad, "k1s")


# -------------------------------------------------- vector kernel KATs
def test_bound_dual_recovery():
    """test_kkt.cpp:335-348"""
    L = O.orc()
    x, lb, ub = np.array([0.5]), np.array([0.0]), np.array([1.0])
    zl, zu, dx = np.array([2.0]), np.array([3.0]), np.array([0.25])
    dzl, dzu = np.zeros(1), np.zeros(1)
    L.orc_recover_bound_duals(1, O._dp_(x), O._dp_(lb), O._dp_(ub), O._dp_(zl), O._dp_(zu), 0.1,
                              O._dp_(dx), O._dp_(dzl), O._dp_(dzu))
    assert abs(dzl[0] + 2.8) <= 1e-14 * 2.8 and abs(dzu[0] + 1.3) <= 1e-14 * 1.3
    lb[0], ub[0] = -np.inf, np.inf
    L.orc_recover_bound_duals(1, O._dp_(x), O._dp_(lb), O._dp_(ub), O._dp_(zl), O._dp_(zu), 0.1,
                              O._dp_(dx), O._dp_(dzl), O._dp_(dzu))
    assert dzl[0] == 0.0 and dzu[0] == 0.0


def test_barrier_residual_blocks():
    """test_kkt.cpp:350-375"""
    L = O.orc()
    f = lambda *v: np.array(v, float)
    jp_ptr, jp_idx = np.array([0, 1], np.int32), np.array([0], np.int32)
    out = np.zeros(5)
    stat, mult, prim, cl, cu = (np.zeros(1) for _ in range(5))
    L.orc_barrier_kkt_residual(1, 0, 1, O._ip_(jp_ptr), O._ip_(jp_idx), O._dp_(f(2.0)),
                               O._dp_(f(1.5)), O._dp_(f(0.2)), O._dp_(f(-0.1)), O._dp_(f(0.7)),
                               O._dp_(f(0.3)), 100.0, O._dp_(f(2.0)), O._dp_(f(0.0)),
                               O._dp_(f(np.inf)), O._dp_(f(0.3)), O._dp_(f(0.0)), 0.5,
                               O._dp_(stat), O._dp_(mult), O._dp_(prim), O._dp_(cl), O._dp_(cu),
                               O._dp_(out))
    assert abs(stat[0] + 0.2) <= 1e-14 * 0.2
    assert abs(mult[0] + 10.4) <= 1e-13 * 10.4
    assert abs(prim[0] - 0.1) <= 1e-14 * 0.1
    assert abs(cl[0] - 0.1) <= 1e-14 * 0.1 and cu[0] == 0.0
    assert abs(out.max() - 10.4) <= 1e-13 * 10.4


def test_fraction_to_boundary():
    """test_ipm.cpp:166-186"""
    L = O.orc()
    f = lambda *v: np.array(v, float)
    ftb = lambda x, lb, ub, dx, tau: L.orc_fraction_to_boundary(len(x), O._dp_(f(*x)), O._dp_(f(*lb)),
                                                                 O._dp_(f(*ub)), O._dp_(f(*dx)), tau)
    assert ftb([0.5], [0.0], [1.0], [-1.0], 0.99) == 0.495
    assert abs(ftb([0.9], [0.0], [1.0], [1.0], 0.99) - 0.099) <= 1e-12
    assert ftb([0.5], [0.0], [1.0], [0.3], 0.99) == 1.0
    z = f(1.0, 0.0)
    assert L.orc_dual_fraction_to_boundary(2, O._dp_(z), O._dp_(f(-2.0, -5.0)), 0.99) == 0.495
    assert L.orc_dual_fraction_to_boundary(2, O._dp_(z), O._dp_(f(2.0, 5.0)), 0.99) == 1.0


def test_outer_schedule_chain():
    """test_solver.cpp:35-71"""
    L = O.orc()
    s = np.zeros(5)
    L.orc_initial_outer_state(0.1, 100.0, 1e14, O._dp_(s))
    assert abs(s[1] - 0.0794328234724) <= 1e-12
    assert abs(s[2] - 8.91250938134) <= 1e-10
    assert L.orc_outer_update(O._dp_(s), 0.0) == 1
    assert abs(s[0] - 0.0102329299228) <= 1e-12
    rho = s[3]
    for _ in range(20):
        assert L.orc_outer_update(O._dp_(s), 1e9) == 0
    assert s[3] == 1e14 and rho == 100.0
