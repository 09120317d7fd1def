"""Accuracy diagnostic: GPU KKT solve vs the oracle (delta loop, refinement
counts, residuals, step error).  python tools/kkt_accuracy.py <spec>..."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from helpers import problem_from_instance, case_from_dict, gpu_context, gpu_input
from oracle import oracle as O
from paper_2510_05885_b200 import instances as I
for spec in sys.argv[1:]:
    inst = I.build(spec); prob = problem_from_instance(inst)
    case = case_from_dict(I.kkt_case(inst, 42))
    for form in ("k2r", "k1s"):
        g = gpu_context(prob, form).solve(gpu_input(case), 0.0)
        Q = O.OrcKkt(prob, form); o = Q.solve(case, 0.0)
        o0 = O.OrcKkt(prob, form, (1e-10, 0, 1e-12, 1e40, 1e-8)).solve(case, 0.0)
        g0c = gpu_context(prob, form, opts=(1e-10, 0, 1e-12, 1e40, 1e-8)) if False else None
        sc = max(1.0, np.abs(o.dx).max(), np.abs(o.dy).max())
        err = max(np.abs(g.dx - o.dx).max(), np.abs(g.dy - o.dy).max()) / sc
        print(f"{spec} {form}: delta {g.delta:.3g}/{o.delta:.3g} att {g.factor_attempts}/{o.factor_attempts} "
              f"refine {g.refine_steps}/{o.refine_steps} rel {g.rel_residual:.2e}/{o.rel_residual:.2e} ref r0 {o0.rel_residual:.2e} step err {err:.2e}", flush=True)
