"""Ad-hoc GPU check used during development (not collected by pytest)."""
import sys, time, traceback
sys.path.insert(0, '/root/repo')
import numpy as np
from oracle import oracle as O
import paper_2510_05885_b200 as P

specs = sys.argv[1:] or ["hs35", "opf-toy-30", "opf-toy-1000", "ncvx-qp-200", "elec:20:3", "bearing:20:20",
                         "opf_mesh:20:20:7", "mpcc_sep:200", "opf_toy:5000:1", "opf_mesh:70:70:1"]
for spec in specs:
    M = O.RefModel(spec); pr = M.problem
    for form, fi in [("k2r", 1), ("k1s", 2), ("k2", 0)]:
        if form == "k2" and pr.n + 2 * pr.m > 5000:
            continue
        try:
            c = M.kkt_case(42)
            hp = P.HessianPattern(pr.nt, pr.hp_ptr, pr.hp_idx); jp = P.JacobianPattern(pr.m, pr.nt, pr.jp_ptr, pr.jp_idx)
            ctx = P.KktContext(hp, jp, pr.nt, pr.ns, pr.m_eq, P.KktForm(fi))
            inp = P.KktInput(c.hval, c.jval, c.sigma, c.rbar1, c.rbar2, c.rbar3, c.rho)
            Q = O.OrcKkt(pr, form)
            Kg = ctx.refill(inp, 0.0); Ko = Q.refill(c, 0.0)
            kbit = np.array_equal(Kg.view(np.int64), Ko.view(np.int64))
            t0 = time.time(); sg = ctx.solve(inp, 0.0); t1 = time.time()
            so = Q.solve(c, 0.0); t2 = time.time()
            fg = ctx.factors(); fo = Q.last_factors()
            sc = max(1.0, np.abs(so.dx).max() if len(so.dx) else 1.0)
            err = max([np.abs(sg.dx - so.dx).max() if len(so.dx) else 0, np.abs(sg.dy - so.dy).max() if len(so.dy) else 0,
                       np.abs(sg.dr - so.dr).max() if len(so.dr) else 0]) / sc if sg.ok else -1
            derr = np.abs(fg['d'] - fo['d']).max() / max(1, np.abs(fo['d']).max())
            lerr = np.abs(fg['lval'] - fo['lval']).max() if len(fo['lval']) else 0
            lri = np.array_equal(fg['lrow_ind'], fo['lrow_ind'])
            print(f"{spec:18s} {form:4s} K_bitexact={kbit} ok={sg.ok}/{so.ok} att={sg.factor_attempts}/{so.factor_attempts} "
                  f"ref={sg.refine_steps}/{so.refine_steps} pert={sg.perturbed_pivots}/{so.perturbed_pivots} "
                  f"inertia={fg['n_pos']},{fg['n_neg']}/{fo['n_pos']},{fo['n_neg']} lrow={lri} derr={derr:.1e} lerr={lerr:.1e} "
                  f"step_err={err:.2e} t_gpu={1e3*(t1-t0):.2f}ms t_cpu={1e3*(t2-t1):.2f}ms", flush=True)
        except Exception:
            traceback.print_exc()
