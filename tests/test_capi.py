"""C-ABI boundary (include/ncl_b200.h) without a GPU: the library loads, exports
every declared symbol, and its host-side symbolic analysis is bit-exact with
the oracle (and therefore with the reference: test_pinning.py)."""
import os
import re

import numpy as np
import pytest

import paper_2510_05885_b200 as P
from helpers import golden_kkt_files, load_golden, problem_from_instance
from oracle import oracle as O
from paper_2510_05885_b200 import _lib
from paper_2510_05885_b200 import instances as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ncl_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ncl_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_kkt_boundary():
    syms = declared_symbols()
    for s in ("ncl_kkt_create", "ncl_kkt_solve", "ncl_kkt_solve_device", "ncl_kkt_symbolic",
              "ncl_kkt_matrix", "ncl_kkt_destroy", "ncl_sparse_factorize", "ncl_sparse_solve_refined"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    # and the ctypes signature table covers them all
    assert set(declared_symbols()) <= set(_lib.SIGS)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def plan_of(prob, form):
    hp = P.HessianPattern(prob.nt, prob.hp_ptr, prob.hp_idx)
    jp = P.JacobianPattern(prob.m, prob.nt, prob.jp_ptr, prob.jp_idx)
    return P.KktPlan(hp, jp, prob.nt, prob.ns, prob.m_eq, P.parse_kkt_form(form))


@pytest.mark.parametrize("path", golden_kkt_files(), ids=lambda p: os.path.basename(p)[4:-4])
def test_host_symbolic_matches_reference_fixture(path):
    z, prob, _ = load_golden(path)
    for form in ("k2", "k2r", "k1s"):
        pl = plan_of(prob, form)
        cp, ri = pl.pattern()
        assert np.array_equal(cp, z[f"{form}_K_colptr"]) and np.array_equal(ri, z[f"{form}_K_rowind"])
        sym = pl.symbolic()
        for k in ("perm", "parent", "lcol_ptr"):
            assert np.array_equal(sym[k], z[f"{form}_{k}"]), (form, k)


@pytest.mark.parametrize("spec", ["opf_toy:4000:3", "opf_mesh:40:30:2", "mpcc_sep:500",
                                  "opf_toy:11:1", "opf_mesh:1:5:1"])
def test_host_symbolic_matches_oracle_on_generated(spec):
    prob = problem_from_instance(I.build(spec))
    for form in ("k2r", "k1s"):
        pl = plan_of(prob, form)
        Q = O.OrcKkt(prob, form)
        a, b = pl.symbolic(), Q.symbolic()
        for k in ("perm", "parent", "lcol_ptr"):
            assert np.array_equal(a[k], b[k]), (form, k)
        assert pl.info.l_nnz == b["lcol_ptr"][-1]


def test_analyze_host_matches_oracle_random_patterns():
    rng = np.random.default_rng(5)
    for n in (1, 2, 17, 60, 300):
        k = 3 * n
        r = rng.integers(0, n, k)
        c = rng.integers(0, n, k)
        r = np.concatenate([r, np.arange(n)])
        c = np.concatenate([c, np.arange(n)])
        got = P.analyze_host(n, r, c)
        S = O.OrcSparse(n, r, c, np.ones(len(r)))
        want = S.symbolic()
        for key in ("perm", "parent", "lcol_ptr"):
            assert np.array_equal(got[key], want[key])
        # explicit permutation path (analyze_with_permutation)
        perm = rng.permutation(n)
        got = P.analyze_host(n, r, c, perm)
        want = O.OrcSparse(n, r, c, np.ones(len(r)), perm).symbolic()
        for key in ("perm", "parent", "lcol_ptr"):
            assert np.array_equal(got[key], want[key])


def test_structural_diagonal_rule_dense_absorption():
    """Eigen's AMD absorbs nodes without a structural diagonal into the dummy
    root (ordered last): K2's y-block (kkt.cpp:85-88) exercises it."""
    n = 6
    rows = [0, 1, 2, 3, 4, 5, 3]
    cols = [0, 1, 2, 0, 1, 2, 3]  # 4, 5 have no diagonal? (5,2),(4,1) + diag present
    rows = [0, 1, 2, 3, 4, 5]
    cols = [0, 1, 2, 0, 1, 2]     # nodes 3,4,5 lack diagonals
    got = P.analyze_host(n, rows, cols)
    want = O.OrcSparse(n, rows, cols, np.ones(len(rows))).symbolic()
    assert np.array_equal(got["perm"], want["perm"])
    assert set(got["perm"][-3:]) == {3, 4, 5}


def test_invalid_arguments_raise_like_the_reference():
    prob = problem_from_instance(I.build("opf_toy:20:1"))
    hp = P.HessianPattern(prob.nt, prob.hp_ptr, prob.hp_idx)
    jp = P.JacobianPattern(prob.m, prob.nt, prob.jp_ptr, prob.jp_idx)
    with pytest.raises(ValueError):   # ns != m - m_eq  (kkt.cpp:52-53)
        P.KktPlan(hp, jp, prob.nt, prob.ns + 1, prob.m_eq, P.KktForm.K1s)
    with pytest.raises(ValueError):   # unknown form (kkt.cpp:13)
        P.parse_kkt_form("k4")
    with pytest.raises(ValueError):   # triplet index out of range (sparse.cpp:43)
        P.analyze_host(3, [0, 5], [0, 1])
    with pytest.raises(ValueError):   # not a permutation (sparse.cpp:115)
        P.analyze_host(3, [0, 1, 2], [0, 1, 2], perm=[0, 0, 1])
    bad = jp.idx.copy()
    bad[0], bad[1] = bad[1], bad[0]   # unsorted Jacobian row
    with pytest.raises(ValueError):
        P.KktPlan(hp, P.JacobianPattern(jp.rows, jp.cols, jp.ptr, bad), prob.nt, prob.ns, prob.m_eq,
                  P.KktForm.K1s)


def test_compute_fails_loudly_without_gpu(monkeypatch):
    """No CPU fallback: with no device visible the product raises."""
    L = _lib.lib()
    if L.ncl_device_count() > 0:
        pytest.skip("a GPU is visible")
    prob = problem_from_instance(I.build("opf_toy:20:1"))
    with pytest.raises(_lib.NclError):
        P.KktContext(P.HessianPattern(prob.nt, prob.hp_ptr, prob.hp_idx),
                     P.JacobianPattern(prob.m, prob.nt, prob.jp_ptr, prob.jp_idx),
                     prob.nt, prob.ns, prob.m_eq, P.KktForm.K1s)
