"""Full NCL solve time (BASELINE metric, first half): the reference's own
driver (proj/src, compiled unmodified) on its CPU KktContext vs the same
driver on the B200 KktContext (integration/ drop-in build), same instance,
form and tolerance.  One host core each.

    python tools/ncl_solve_time.py <spec> <form> [tol] [--device-init]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from integration import drop  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    spec, form = args[0], args[1]
    tol = float(args[2]) if len(args) > 2 else 1e-8
    if "--device-init" in sys.argv:
        os.environ["NCL_B200_INIT_MULTIPLIERS"] = "1"
    g_model = drop.DropModel(spec)
    g_model.solve(form=form, tol=tol, max_outer=1, max_inner=2)  # warm-up: CUDA context, graphs
    t0 = time.perf_counter()
    g = g_model.solve(form=form, tol=tol)
    tg = time.perf_counter() - t0
    line = (f"{spec} {form} tol {tol:g}: B200 drop-in {g['status']} outer {g['outer_iters']} inner "
            f"{g['inner_iters']} solve {g['solve_seconds']:.3f}s (wall {tg:.3f}s) obj {g['objective']:.12g}")
    if "--no-ref" not in sys.argv:
        t0 = time.perf_counter()
        r = O.RefModel(spec).solve(form=form, tol=tol)
        tr = time.perf_counter() - t0
        rel = abs(g["objective"] - r["objective"]) / max(1.0, abs(r["objective"]))
        line += (f" | reference CPU {r['status']} outer {r['outer_iters']} inner {r['inner_iters']} solve "
                 f"{r['solve_seconds']:.3f}s (wall {tr:.3f}s) | speed-up {r['solve_seconds'] / g['solve_seconds']:.1f}x"
                 f" | objective rel diff {rel:.1e}")
    print(line, flush=True)


if __name__ == "__main__":
    main()
