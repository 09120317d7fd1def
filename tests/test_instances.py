"""The numpy instance generators (paper_2510_05885_b200/instances.py) against
the reference's own Model (golden fixtures always; live reference when built):
identical patterns and bounds, derivative values to rounding."""
import os
import subprocess

import numpy as np
import pytest

from helpers import GOLDEN
from oracle import oracle as O
from paper_2510_05885_b200 import instances as I

PAIRS = [("opf-toy-30", "opf_toy:15:201"), ("opf-toy-200", "opf_toy:100:202"),
         ("mpcc-sep-50", "mpcc_sep:25"), ("opf_mesh:8:8:3", "opf_mesh:8:8:3")]


def test_mt19937_64_matches_libstdcxx_known_values():
    # std::mt19937_64 default seed 5489: the 10000th output is 9981545732273789042
    g = I.MT19937_64(5489)
    assert int(g.raw(10000)[-1]) == 9981545732273789042


@pytest.mark.parametrize("ref_name,spec", PAIRS)
def test_generator_matches_reference_fixture(ref_name, spec):
    z = np.load(os.path.join(GOLDEN, f"kkt_{ref_name.replace(':', '_').replace('-', '_')}.npz"))
    inst = I.build(spec)
    for k in ("hp_ptr", "hp_idx", "jp_ptr", "jp_idx"):
        assert np.array_equal(getattr(inst, k), z[k]), k
    assert (inst.nt, inst.ns, inst.m_eq, inst.m) == (int(z["nt"]), int(z["ns"]), int(z["m_eq"]), int(z["m"]))
    assert np.array_equal(inst.lb, z["lb"]) and np.array_equal(inst.ub, z["ub"])
    assert np.array_equal(inst.start, z["start"])
    c = I.kkt_case(inst, 42)
    for k in ("sigma", "rbar1", "rbar2", "rbar3"):
        assert np.array_equal(c[k], z[k]), k
    for k in ("hval", "jval"):
        assert np.abs(c[k] - z[k]).max() <= 1e-14 * max(1.0, np.abs(z[k]).max()), k


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("spec", ["opf_toy:2000:5", "opf_mesh:31:17:4", "mpcc_sep:300", "elec:40:5"])
def test_generator_matches_live_reference(spec):
    M = O.RefModel(spec)
    inst = I.build(spec)
    p = M.problem
    for k in ("hp_ptr", "hp_idx", "jp_ptr", "jp_idx"):
        assert np.array_equal(getattr(inst, k), getattr(p, k)), k
    assert np.array_equal(inst.lb, p.lb) and np.array_equal(inst.ub, p.ub)
    c, r = I.kkt_case(inst, 7), M.kkt_case(7)
    for k in ("hval", "jval"):
        assert np.abs(c[k] - getattr(r, k)).max() <= 1e-13 * max(1.0, np.abs(getattr(r, k)).max())


def test_mesh_is_bushier_than_ring():
    """the perf variant of SURVEY.md 8(d): far shallower elimination tree"""
    import paper_2510_05885_b200 as P
    from helpers import problem_from_instance

    def height(spec):
        prob = problem_from_instance(I.build(spec))
        pl = P.KktPlan(P.HessianPattern(prob.nt, prob.hp_ptr, prob.hp_idx),
                       P.JacobianPattern(prob.m, prob.nt, prob.jp_ptr, prob.jp_idx),
                       prob.nt, prob.ns, prob.m_eq, P.KktForm.K1s)
        return pl.info.sn_height

    assert height("opf_mesh:60:60:1") * 20 < height("opf_toy:3600:1")


def test_bearing_is_a_weighted_5_point_stencil():
    """COPS bearing (repo generator): lower CSC with
    sorted rows, m = 0, symmetric positive definite Hessian"""
    import scipy.sparse as sp
    inst = I.build("bearing:9:7")
    n = inst.nt
    assert (inst.m, inst.m_eq, inst.ns) == (0, 0, 0) and n == 63
    for c in range(n):
        rows = inst.hp_idx[inst.hp_ptr[c]:inst.hp_ptr[c + 1]]
        assert rows[0] == c and np.all(np.diff(rows) > 0) and set(rows[1:]) <= {c + 1, c + 9}
    h, jv, g, cv = inst.evaluator.eval(np.ones(n), np.zeros(0))
    assert len(jv) == 0 and len(cv) == 0
    L = sp.csc_matrix((h, inst.hp_idx, inst.hp_ptr), shape=(n, n))
    A = (L + L.T - sp.diags(L.diagonal())).toarray()
    assert np.allclose(A, A.T) and np.linalg.eigvalsh(A).min() > 0
    assert np.allclose(g, A @ np.ones(n) + np.tile(inst.evaluator.lin, 7))
