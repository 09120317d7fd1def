"""Generate the golden fixtures from the REFERENCE itself.

Run in the container that has /root/reference (the reference library is
compiled unmodified from proj/src against oracle/eigen_shim by
``make -C oracle ref``):

    python tests/golden/make_golden.py

Writes tests/golden/kkt_<instance>.npz: the instance patterns, the
test_kkt.cpp:40-68 input recipe evaluated by the reference's own AD, and for
every KKT form the reference KktContext's outputs (assembled K, step, stats)
plus the reference's symbolic analysis of K.  Also writes
tests/golden/solve_<instance>.npz with full NCL solve reports (iteration
logs) for end-to-end checks.  The fixtures travel with the repo; the GPU box
never needs /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

KKT_INSTANCES = ["hs35", "hs6", "hs7", "redundant-circle", "dup-rows", "opf-toy-30", "opf-toy-200",
                 "mpcc-sep-50", "ncvx-qp-50", "convex-qp-50", "mpcc-basic", "elec:12:3",
                 "bearing:8:8", "opf_mesh:8:8:3"]
SOLVE_INSTANCES = [("hs35", "k1s"), ("hs35", "k2r"), ("hs7", "k2r"), ("opf-toy-30", "k1s"),
                   ("opf-toy-30", "k2r"), ("mpcc-basic", "k2r"), ("mpcc-sep-10", "k2r"),
                   ("dup-rows", "k1s"), ("rosenbrock-box", "k1s")]


def fname(spec):
    return spec.replace(":", "_").replace("-", "_")


def main():
    O.build(ref=True)
    for spec in KKT_INSTANCES:
        M = O.RefModel(spec)
        p = M.problem
        c = M.kkt_case(42)
        out = dict(nt=p.nt, ns=p.ns, m_eq=p.m_eq, m=p.m, hp_ptr=p.hp_ptr, hp_idx=p.hp_idx,
                   jp_ptr=p.jp_ptr, jp_idx=p.jp_idx, lb=p.lb, ub=p.ub, start=p.start,
                   hval=c.hval, jval=c.jval, sigma=c.sigma, rbar1=c.rbar1, rbar2=c.rbar2,
                   rbar3=c.rbar3, rho=c.rho)
        for form in ("k2", "k2r", "k1s"):
            R = O.RefKkt(p, form)
            s = R.solve(c, 0.0)
            cp, ri, v = R.matrix()
            rows = np.repeat(np.arange(R.N), np.diff(cp))
            # the reference's analyze() of K (sparse.cpp:178-180)
            sp_h = O.ref().ref_sparse_new(R.N, len(ri), O._ip_(O.i32(ri)), O._ip_(O.i32(rows)),
                                          O._dp_(O.f64(v)), None)
            perm = np.zeros(R.N, np.int32)
            parent = np.zeros(R.N, np.int32)
            lcp = np.zeros(R.N + 1, np.int32)
            amap = np.zeros(len(ri), np.int32)
            O.ref().ref_sparse_symbolic(sp_h, O._ip_(perm), O._ip_(parent), O._ip_(lcp), O._ip_(amap))
            O.ref().ref_sparse_free(sp_h)
            out.update({f"{form}_K_colptr": cp, f"{form}_K_rowind": ri, f"{form}_K_val": v,
                        f"{form}_dx": s.dx, f"{form}_dr": s.dr, f"{form}_dy": s.dy,
                        f"{form}_stats": np.array([s.delta, s.factor_attempts, s.refine_steps,
                                                   s.perturbed_pivots, s.rel_residual, s.ok]),
                        f"{form}_perm": perm, f"{form}_parent": parent, f"{form}_lcol_ptr": lcp})
        np.savez_compressed(os.path.join(HERE, f"kkt_{fname(spec)}.npz"), **out)
        print("wrote", spec)
    for spec, form in SOLVE_INSTANCES:
        M = O.RefModel(spec)
        r = M.solve(form=form, tol=1e-8)
        np.savez_compressed(os.path.join(HERE, f"solve_{fname(spec)}_{form}.npz"),
                            status=r["status"], objective=r["objective"],
                            kkt_residual=r["kkt_residual"], primal_feas=r["primal_feas"],
                            outer_iters=r["outer_iters"], inner_iters=r["inner_iters"],
                            log=r["log"], extrap_alpha=r["extrap_alpha"], x=r["x"], y=r["y"])
        print("wrote solve", spec, form, r["status"], r["objective"])


if __name__ == "__main__":
    main()
