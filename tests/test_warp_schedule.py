"""Host-side invariants of the warp-tier schedule (csrc/symbolic.cpp), checked
through the C ABI without a GPU (ncl_plan_check_schedule):

* every warp-tier node on exactly one path, each path a child -> parent chain;
* hand-out order of the persistent kernels: the long root paths first (tops
  without a warp-tier parent, so nothing waits on them), every other path
  after the paths of all its light children (no warp spins on unstarted work);
* the backward solve's order: each path after the path of its top's parent;
* light-child extend-add chunks: 32 entries, destinations distinct within a
  chunk, exactly the light children's update entries, per destination in
  child order (deterministic sums);
* the per-path-position node records agree with the supernodal arrays.

Both the plan's own structure (the reference's postorder) and the
re-postordered one the device factorization uses (tallest child last, relaxed
warp-tier supernodes) are checked."""
import numpy as np
import pytest

import paper_2510_05885_b200 as P
from paper_2510_05885_b200 import _lib
from paper_2510_05885_b200 import instances as I
from helpers import problem_from_instance


def plan(spec, form):
    prob = problem_from_instance(I.build(spec))
    return P.KktPlan(P.HessianPattern(prob.nt, prob.hp_ptr, prob.hp_idx),
                     P.JacobianPattern(prob.m, prob.nt, prob.jp_ptr, prob.jp_idx),
                     prob.nt, prob.ns, prob.m_eq, P.parse_kkt_form(form))


@pytest.mark.parametrize("spec,form", [
    ("opf_toy:3000:1", "k1s"),      # ring: chain-shaped tree, front paths
    ("opf_toy:3000:2", "k2r"),
    ("opf_mesh:30:30:1", "k1s"),    # grid: warp tier under a wide tier
    ("opf_mesh:12:9:3", "k2"),
    ("mpcc_sep:500", "k2r"),        # many tiny independent trees
    ("elec:60:1", "k2r"),           # dense block: everything wide
    ("bearing:40:30", "k2r"),       # 2-D grid, no constraints
])
@pytest.mark.parametrize("internal", [0, 1])
def test_warp_schedule_invariants(spec, form, internal):
    pl = plan(spec, form)
    rc = _lib.lib().ncl_plan_check_schedule(pl._h, internal)
    assert rc == 0, _lib.lib().ncl_last_error().decode()


def test_ring_has_a_front_path():
    """the reference generator's ring at 3000 buses: one chain long enough to
    be handed out first (>= 64 warp-tier nodes) -- the case the front-path
    order exists for"""
    pl = plan("opf_toy:3000:1", "k1s")
    assert pl.info.sn_height >= 64
    assert pl.info.n_wide == 0
