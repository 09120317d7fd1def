"""init_multipliers (proj/src/solver.cpp:43-91) on the device: SURVEY.md 8(f)
row 1.  The candidate pairs replace the reference's all-pairs loop (:55-79);
the kept triplets, their values and the factorization settings are the
reference's, so the multipliers match the C restatement (itself pinned to the
reference library, tests/test_pinning.py) to rounding."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_05885_b200 import _lib
from paper_2510_05885_b200 import instances as I


def candidates(inst):
    L = _lib.lib()
    cnt = C.c_longlong()
    jp = np.ascontiguousarray(inst.jp_ptr, np.int32)
    ji = np.ascontiguousarray(inst.jp_idx, np.int32)
    _lib.check(L.ncl_jjt_candidates(inst.m, inst.nt, _lib.ip(jp), _lib.ip(ji), 0, C.byref(cnt), None, None),
               "ncl_jjt_candidates")
    pi = np.zeros(cnt.value, np.int32)
    pj = np.zeros(cnt.value, np.int32)
    _lib.check(L.ncl_jjt_candidates(inst.m, inst.nt, _lib.ip(jp), _lib.ip(ji), cnt.value, C.byref(cnt),
                                    _lib.ip(pi), _lib.ip(pj)), "ncl_jjt_candidates")
    return pi, pj


@pytest.mark.parametrize("spec", ["opf_toy:60:3", "opf_mesh:6:5:2", "mpcc_sep:40"])
def test_candidate_pairs_are_the_rows_sharing_a_column(spec):
    """the reference keeps (i, j <= i) iff i == j or the dot is nonzero; a
    nonzero dot needs a shared column, so these pairs cover every kept one"""
    inst = I.build(spec)
    pi, pj = candidates(inst)
    rows = [set(inst.jp_idx[inst.jp_ptr[i]:inst.jp_ptr[i + 1]].tolist()) for i in range(inst.m)]
    want = [(i, j) for i in range(inst.m) for j in range(i + 1) if i == j or rows[i] & rows[j]]
    assert list(zip(pi.tolist(), pj.tolist())) == want


def oracle_y(inst, jval, g):
    y = np.zeros(inst.m)
    O.orc().orc_init_multipliers(inst.m, inst.m_eq, O._ip_(O.i32(inst.jp_ptr)), O._ip_(O.i32(inst.jp_idx)),
                                 O._dp_(O.f64(jval)), O._dp_(O.f64(g)), O._dp_(y))
    return y


def device_y(inst, jval, g):
    L = _lib.lib()
    y = np.zeros(inst.m)
    sec = np.zeros(4)
    jp = np.ascontiguousarray(inst.jp_ptr, np.int32)
    ji = np.ascontiguousarray(inst.jp_idx, np.int32)
    _lib.check(L.ncl_init_multipliers(inst.m, inst.m_eq, inst.nt, _lib.ip(jp), _lib.ip(ji), _lib.dp(jval),
                                      _lib.dp(g), _lib.dp(y), _lib.dp(sec)), "ncl_init_multipliers")
    return y, sec


@pytest.mark.gpu
@pytest.mark.parametrize("spec", ["opf_toy:3000:7", "opf_mesh:30:30:3", "mpcc_sep:2000", "opf_toy:11:2"])
def test_gpu_init_multipliers_matches_oracle(spec):
    inst = I.build(spec)
    rng = I.MT19937_64(17)
    t = inst.start + rng.uniform(-0.05, 0.05, inst.nt)
    _, jval, grad, _ = inst.evaluator.eval(t, np.zeros(inst.m))
    yo = oracle_y(inst, jval, grad)
    yg, sec = device_y(inst, np.ascontiguousarray(jval), np.ascontiguousarray(grad))
    assert np.all(np.abs(yg) <= 1e3)
    assert np.abs(yg - yo).max() <= 1e-8 * max(1.0, np.abs(yo).max())
