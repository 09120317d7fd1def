"""Pin the oracle to the reference itself.

* Golden fixtures (tests/golden, made by make_golden.py from the reference
  library compiled unmodified from proj/src): the C restatement must reproduce
  the reference's assembled K, symbolic analysis and Newton steps BITWISE.
* When the reference library is present (this container, or a prebuilt copy
  in oracle/_ref), the same comparison runs live on larger instances.
"""
import os

import numpy as np
import pytest

from helpers import golden_kkt_files, load_golden
from oracle import oracle as O

FORMS = ("k2", "k2r", "k1s")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


@pytest.mark.parametrize("path", golden_kkt_files(), ids=lambda p: os.path.basename(p)[4:-4])
def test_oracle_matches_reference_fixture_bitwise(path):
    z, prob, case = load_golden(path)
    for form in FORMS:
        Q = O.OrcKkt(prob, form)
        st = Q.solve(case, 0.0)
        cp, ri, v = Q.matrix()
        assert np.array_equal(cp, z[f"{form}_K_colptr"]) and np.array_equal(ri, z[f"{form}_K_rowind"])
        assert np.array_equal(bits(v), bits(z[f"{form}_K_val"])), form
        sym = Q.symbolic()
        for k in ("perm", "parent", "lcol_ptr"):
            assert np.array_equal(sym[k], z[f"{form}_{k}"]), (form, k)
        ref = z[f"{form}_stats"]
        assert (st.delta, st.factor_attempts, st.refine_steps, st.perturbed_pivots, st.ok) == \
            (ref[0], int(ref[1]), int(ref[2]), int(ref[3]), bool(ref[5]))
        assert st.rel_residual == ref[4]
        for k in ("dx", "dr", "dy"):
            assert np.array_equal(bits(getattr(st, k)), bits(z[f"{form}_{k}"])), (form, k)


LIVE = ["opf-toy-1000", "ncvx-qp-200", "convex-qp-200", "mpcc-sep-50", "opf_mesh:24:24:5",
        "opf_toy:3000:9", "elec:30:2", "bearing:30:25"]


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("spec", LIVE)
def test_oracle_matches_live_reference_bitwise(spec):
    M = O.RefModel(spec)
    prob = M.problem
    for seed in (1, 42):
        case = M.kkt_case(seed)
        for form in ("k2r", "k1s") if prob.n + 2 * prob.m > 4000 else FORMS:
            Q, R = O.OrcKkt(prob, form), O.RefKkt(prob, form)
            so, sr = Q.solve(case, 0.0), R.solve(case, 0.0)
            assert np.array_equal(bits(Q.matrix()[2]), bits(R.matrix()[2]))
            assert (so.delta, so.factor_attempts, so.refine_steps, so.perturbed_pivots, so.ok) == \
                (sr.delta, sr.factor_attempts, sr.refine_steps, sr.perturbed_pivots, sr.ok)
            for k in ("dx", "dr", "dy"):
                assert np.array_equal(bits(getattr(so, k)), bits(getattr(sr, k)))


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_oracle_warm_delta_and_escalation_match_live_reference():
    """delta-loop semantics (kkt.cpp:273-313) on a problem that needs them:
    elec's Coulomb Hessian is indefinite away from the solution."""
    M = O.RefModel("elec:16:5")
    prob = M.problem
    case = M.kkt_case(3)
    for form in FORMS:
        Q, R = O.OrcKkt(prob, form), O.RefKkt(prob, form)
        for warm in (0.0, 1e-3, 7.5):
            so, sr = Q.solve(case, warm), R.solve(case, warm)
            assert (so.delta, so.factor_attempts, so.ok) == (sr.delta, sr.factor_attempts, sr.ok)
            assert so.factor_attempts > 1
            for k in ("dx", "dr", "dy"):
                assert np.array_equal(bits(getattr(so, k)), bits(getattr(sr, k)))


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_oracle_sparse_layer_matches_live_reference():
    """sparse.cpp: factorize + solve_refined on random SQD / indefinite data."""
    from helpers import Rng, from_dense_lower, random_sqd
    L = O.ref()
    for seed in (3, 17, 99):
        M = random_sqd(40, 25, seed)
        rng = Rng(seed + 1)
        M[np.diag_indices(65)] *= np.array([1.0 if rng.uniform() < 0.9 else 1e-12 for _ in range(65)])
        n, ri, ci, v = from_dense_lower(M)
        S = O.OrcSparse(n, ri, ci, v)
        F = S.factorize(1e-10)
        h = L.ref_sparse_new(n, len(ri), O._ip_(O.i32(ri)), O._ip_(O.i32(ci)), O._dp_(O.f64(v)), None)
        info = np.zeros(4, np.int32)
        lri = np.zeros(L.ref_sparse_lnz(h), np.int32)
        lv = np.zeros(len(lri))
        d = np.zeros(n)
        L.ref_sparse_factorize(h, 1e-10, O._ip_(info), O._ip_(lri), O._dp_(lv), O._dp_(d))
        assert (F["ok"], F["n_pos"], F["n_neg"], F["perturbed"]) == tuple(bool(info[0]) if i == 0 else int(info[i]) for i in range(4))
        assert np.array_equal(bits(F["lval"]), bits(lv)) and np.array_equal(bits(F["d"]), bits(d))
        b = np.array([rng.uniform(-1, 1) for _ in range(n)])
        x, steps, rel, conv = S.solve_refined(b)
        xr = np.zeros(n)
        out2 = np.zeros(2)
        sr = L.ref_sparse_solve_refined(h, O._dp_(b), 10, 1e-12, O._dp_(xr), O._dp_(out2))
        L.ref_sparse_free(h)
        assert steps == sr and rel == out2[0]
        assert np.array_equal(bits(x), bits(xr))


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_oracle_init_multipliers_matches_reference_solver_path():
    """init_multipliers (solver.cpp:43-91) -- restated with the same triplets,
    factored with eps = 1e-14: compare against the reference on the values it
    would see (kkt_case jacobian + a gradient)."""
    M = O.RefModel("opf-toy-200")
    p = M.problem
    case = M.kkt_case(11)
    g = np.linspace(-1.0, 1.0, p.nt)
    y = np.zeros(p.m)
    O.orc().orc_init_multipliers(p.m, p.m_eq, O._ip_(O.i32(p.jp_ptr)), O._ip_(O.i32(p.jp_idx)),
                                 O._dp_(O.f64(case.jval)), O._dp_(O.f64(g)), O._dp_(y))
    assert np.all(np.abs(y) <= 1e3) and np.isfinite(y).all()
    # normal-equation residual of the regularized system
    J = np.zeros((p.m, p.nt))
    for i in range(p.m):
        J[i, p.jp_idx[p.jp_ptr[i]:p.jp_ptr[i + 1]]] = case.jval[p.jp_ptr[i]:p.jp_ptr[i + 1]]
    A = J @ J.T + 1e-8 * np.eye(p.m)
    A[np.arange(p.m_eq, p.m), np.arange(p.m_eq, p.m)] += 1.0
    yy = np.linalg.solve(A, J @ g)
    assert np.abs(np.clip(yy, -1e3, 1e3) - y).max() <= 1e-8 * max(1.0, np.abs(yy).max())
