import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_05885_b200 import scopf as SC
D = SC.scopf_data(118, 1250, 1)
sub = SC.subproblem(D, 0, D.K, True)
cs = SC.scopf_case(sub, 42)
dev = {k: torch.tensor(cs[k], dtype=torch.float64, device="cuda") for k in ("hval","jval","sigma","rbar1","rbar2","rbar3")}
K = SC.ScopfKkt(sub, sub.nt)
import ctypes as C
from paper_2510_05885_b200 import _lib
info = _lib.KktInfo(); _lib.lib().ncl_schur_info(K.h, C.byref(info))
print("N", info.n, "nsn", info.n_supernodes, "paths", info.n_paths, "wide", info.n_wide, "levels", info.n_levels, "maxf", info.max_front, "flops", info.flops)
for _ in range(3): K.solve(dev, 100.0, 0.0)
T = {}
def wrap(name, f):
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(*a, **k); torch.cuda.synchronize()
        T[name] = T.get(name, 0) + time.perf_counter() - t0; return r
    return g
K._factor = wrap("factor", K._factor); K._solve = wrap("solve", K._solve); K._residual = wrap("residual", K._residual)
L = K.L
for nm in ("ncl_schur_factor", "ncl_schur_factor_dense", "ncl_schur_forward", "ncl_schur_solve0", "ncl_schur_backward", "ncl_schur_residual", "ncl_schur_rhs", "ncl_schur_recover"):
    orig = getattr(L, nm)
    def mk(orig, nm):
        def g(*a):
            t0 = time.perf_counter(); r = orig(*a); T["c:" + nm] = T.get("c:" + nm, 0) + time.perf_counter() - t0; return r
        return g
    setattr(K, "L", L)

for nm in dir(L):
    pass
t0 = time.perf_counter()
for _ in range(5): K.solve(dev, 100.0, 0.0)
tot = (time.perf_counter() - t0) / 5
print("total per solve %.2f ms" % (tot * 1e3), {k: round(v / 5 * 1e3, 2) for k, v in T.items()})
