"""Parity of this round's wide-tier paths and of their switches, against the
oracle: the tree-dataflow solves (tree_solve.cu; single-CTA and cluster
launches), the panel kernel with the strip update folded in
(k_wide_panel_f), the opt-in persistent huge-level kernel, the mid-front
kernel (single-panel fronts kept in shared memory), the unstaged fallbacks of
the staged gathers, and the kernels they replace.  Every configuration must reach the oracle's decisions and step
(same bars as test_gpu_kkt.py) and be bitwise reproducible from one call to
the next (the second call replays the CUDA graphs).

The switches are read when a context is built, so each configuration builds
its own context with the environment set."""
import os

import numpy as np
import pytest

from helpers import case_from_dict, gpu_context, gpu_input, problem_from_instance
from oracle import oracle as O
from paper_2510_05885_b200 import instances as I
from test_gpu_kkt import STEP_RTOL, check_same_decisions, pre_refinement_residual, step_err

pytestmark = pytest.mark.gpu

CONFIGS = {
    "default": {},
    "level-solves": {"NCL_NO_TREE": "1"},
    "tree-single-cta": {"NCL_TREE_C": "1"},
    "separate-strip": {"NCL_NO_FUSED_PANEL": "1"},
    "persistent-huge": {"NCL_HUGE_LEVEL": "1"},
    "no-mid-fronts": {"NCL_NO_MID": "1"},
    # the mid-front assembly and the tree forward gather without their staged
    # row maps (the paths fronts with more children / entries than the staging
    # buffers hold take)
    "unstaged-gathers": {"NCL_NO_STAGED_GATHER": "1"},
}
SWITCHES = ("NCL_NO_TREE", "NCL_TREE_C", "NCL_NO_FUSED_PANEL", "NCL_HUGE_LEVEL", "NCL_NO_MID", "NCL_NO_STAGED_GATHER")

_cache = {}


def oracle_step(spec, form):
    if (spec, form) not in _cache:
        inst = I.build(spec)
        prob = problem_from_instance(inst)
        case = case_from_dict(I.kkt_case(inst, 42))
        _cache[(spec, form)] = (prob, case, O.OrcKkt(prob, form).solve(case, 0.0))
    return _cache[(spec, form)]


@pytest.mark.parametrize("spec,form", [("opf_mesh:120:120:1", "k1s"), ("opf_mesh:280:280:1", "k1s"),
                                       ("opf_mesh:60:60:1", "k2r")])
@pytest.mark.parametrize("config", sorted(CONFIGS))
def test_gpu_wide_paths_match_oracle(config, spec, form, monkeypatch):
    for k in SWITCHES:
        monkeypatch.delenv(k, raising=False)
    for k, v in CONFIGS[config].items():
        monkeypatch.setenv(k, v)
    prob, case, o = oracle_step(spec, form)
    ctx = gpu_context(prob, form)
    first = ctx.solve(gpu_input(case), 0.0)
    again = ctx.solve(gpu_input(case), 0.0)  # graphs captured / replayed
    check_same_decisions(first, o, borderline=lambda: pre_refinement_residual(prob, form, case))
    assert step_err(first, o) <= STEP_RTOL
    for k in ("dx", "dr", "dy"):
        assert np.array_equal(getattr(first, k).view(np.int64), getattr(again, k).view(np.int64)), k
