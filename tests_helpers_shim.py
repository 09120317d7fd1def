"""Adapter from the numpy instance generators to the oracle's data types
(used by bench.py's CPU-baseline legs only)."""
from oracle import oracle as O


def problem_case(inst, case):
    prob = O.Problem(inst.name, inst.nt, inst.ns, inst.m_eq, inst.m, inst.hp_ptr, inst.hp_idx,
                     inst.jp_ptr, inst.jp_idx, inst.lb, inst.ub, inst.start)
    kc = O.KktCase(case["hval"], case["jval"], case["sigma"], case["rbar1"], case["rbar2"],
                   case["rbar3"], case["rho"])
    return prob, kc
