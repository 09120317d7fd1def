"""Fused NCL vector kernels against the oracle:
bitwise for every vector the reference computes with a defined order, exact
for the max/min reductions."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_05885_b200 import instances as I
from paper_2510_05885_b200 import nlp as N


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def test_outer_schedule_host_kat():
    """test_solver.cpp:35-71 through the C ABI (host function, no GPU)"""
    s = N.initial_outer_state(0.1, 100.0, 1e14)
    assert abs(s[1] - 0.0794328234724) <= 1e-12 and abs(s[2] - 8.91250938134) <= 1e-10
    assert N.outer_update(s, 0.0)
    assert abs(s[0] - 0.0102329299228) <= 1e-12
    for _ in range(20):
        assert not N.outer_update(s, 1e9)
    assert s[3] == 1e14
    # and identical to the restatement on a random sequence of residuals
    a, b = N.initial_outer_state(0.1, 100.0, 1e14), np.zeros(5)
    O.orc().orc_initial_outer_state(0.1, 100.0, 1e14, O._dp_(b))
    rng = np.random.default_rng(3)
    for rn in rng.uniform(0, 0.2, 40) ** 3:
        assert N.outer_update(a, rn) == bool(O.orc().orc_outer_update(O._dp_(b), rn))
        assert np.array_equal(bits(a), bits(b))


def random_state(inst, seed):
    rng = np.random.default_rng(seed)
    n, m = inst.n, inst.m
    lb, ub = inst.lb, inst.ub
    lo = np.where(np.isfinite(lb), lb, -5.0)
    hi = np.where(np.isfinite(ub), ub, 5.0)
    x = lo + (hi - lo) * rng.uniform(0.05, 0.95, n)
    d = dict(x=x, zl=np.where(np.isfinite(lb), rng.uniform(0.01, 2, n), 0.0),
             zu=np.where(np.isfinite(ub), rng.uniform(0.01, 2, n), 0.0),
             grad=rng.uniform(-1, 1, n), c=rng.uniform(-1, 1, m), r=rng.uniform(-.1, .1, m),
             y=rng.uniform(-1, 1, m), yk=rng.uniform(-1, 1, m), dx=rng.uniform(-2, 2, n))
    d["grad"][inst.nt:] = 0.0
    d["jval"] = I.kkt_case(inst, seed)["jval"]
    # exercise zero duals / exact bounds edge cases
    d["zl"][::7] = 0.0
    d["dx"][::5] = 0.0
    return d


SPECS = ["opf_mesh:9:7:2", "opf_toy:300:4", "mpcc_sep:120"]


@pytest.mark.gpu
@pytest.mark.parametrize("spec", SPECS)
def test_vector_kernels_match_oracle_bitwise(spec):
    torch = pytest.importorskip("torch")
    inst = I.build(spec)
    nt, ns, m, n = inst.nt, inst.ns, inst.m, inst.n
    nl = N.Nlp(nt, ns, inst.m_eq, m, inst.jp_ptr, inst.jp_idx, inst.lb, inst.ub)
    L = O.orc()
    for seed in (1, 2):
        st = random_state(inst, seed)
        dv = {k: torch.tensor(v, dtype=torch.float64, device="cuda") for k, v in st.items()}
        z = lambda k: torch.zeros(k, dtype=torch.float64, device="cuda")
        mu, rho = 0.0137, 312.5
        # KktInput (ipm.cpp:184-208)
        sg, r1, r2, r3 = z(n), z(n), z(m), z(m)
        nl.kkt_input(dv["jval"].data_ptr(), dv["grad"].data_ptr(), dv["c"].data_ptr(), dv["x"].data_ptr(),
                     dv["zl"].data_ptr(), dv["zu"].data_ptr(), dv["r"].data_ptr(), dv["y"].data_ptr(),
                     dv["yk"].data_ptr(), mu, rho, sg.data_ptr(), r1.data_ptr(), r2.data_ptr(), r3.data_ptr())
        nl.sync()
        osg, or1, or2, or3 = np.zeros(n), np.zeros(n), np.zeros(m), np.zeros(m)
        P = lambda k: O._dp_(O.f64(st[k]))
        L.orc_kkt_input(nt, ns, m, O._ip_(O.i32(inst.jp_ptr)), O._ip_(O.i32(inst.jp_idx)), P("jval"), P("grad"),
                        P("c"), P("x"), O._dp_(O.f64(inst.lb)), O._dp_(O.f64(inst.ub)), P("zl"), P("zu"),
                        P("r"), P("y"), P("yk"), mu, rho, O._dp_(osg), O._dp_(or1), O._dp_(or2), O._dp_(or3))
        for g, o in ((sg, osg), (r1, or1), (r2, or2), (r3, or3)):
            assert np.array_equal(bits(g.cpu().numpy()), bits(o))
        # barrier residual (kkt.cpp:341-366)
        vs = [z(n), z(m), z(m), z(n), z(n)]
        norms = nl.residual(dv["jval"].data_ptr(), dv["grad"].data_ptr(), dv["c"].data_ptr(), dv["r"].data_ptr(),
                            dv["y"].data_ptr(), dv["yk"].data_ptr(), rho, dv["x"].data_ptr(),
                            dv["zl"].data_ptr(), dv["zu"].data_ptr(), mu, *[t.data_ptr() for t in vs])
        ovs = [np.zeros(n), np.zeros(m), np.zeros(m), np.zeros(n), np.zeros(n)]
        onorm = np.zeros(5)
        L.orc_barrier_kkt_residual(nt, ns, m, O._ip_(O.i32(inst.jp_ptr)), O._ip_(O.i32(inst.jp_idx)), P("jval"),
                                   P("grad"), P("c"), P("r"), P("y"), P("yk"), rho, P("x"),
                                   O._dp_(O.f64(inst.lb)), O._dp_(O.f64(inst.ub)), P("zl"), P("zu"), mu,
                                   *[O._dp_(a) for a in ovs], O._dp_(onorm))
        for g, o in zip(vs, ovs):
            assert np.array_equal(bits(g.cpu().numpy()), bits(o))
        assert np.array_equal(norms, onorm)
        # bound duals + fraction to boundary (kkt.cpp:316-328, ipm.cpp:124-141)
        tau = max(0.99, 1.0 - mu)
        dzl, dzu = z(n), z(n)
        al = nl.step(dv["x"].data_ptr(), dv["zl"].data_ptr(), dv["zu"].data_ptr(), mu, dv["dx"].data_ptr(), tau,
                     dzl.data_ptr(), dzu.data_ptr())
        odzl, odzu = np.zeros(n), np.zeros(n)
        L.orc_recover_bound_duals(n, P("x"), O._dp_(O.f64(inst.lb)), O._dp_(O.f64(inst.ub)), P("zl"), P("zu"),
                                  mu, P("dx"), O._dp_(odzl), O._dp_(odzu))
        assert np.array_equal(bits(dzl.cpu().numpy()), bits(odzl))
        assert np.array_equal(bits(dzu.cpu().numpy()), bits(odzu))
        ap = L.orc_fraction_to_boundary(n, P("x"), O._dp_(O.f64(inst.lb)), O._dp_(O.f64(inst.ub)), P("dx"), tau)
        azl = L.orc_dual_fraction_to_boundary(n, P("zl"), O._dp_(odzl), tau)
        azu = L.orc_dual_fraction_to_boundary(n, P("zu"), O._dp_(odzu), tau)
        assert tuple(al) == (ap, azl, azu)
        # trial step + dual clipping (ipm.cpp:267-279, 232-249)
        xt = z(n)
        nl.axpy(n, dv["x"].data_ptr(), al[0], dv["dx"].data_ptr(), xt.data_ptr())
        nl.sync()
        xt_ref = st["x"] + al[0] * st["dx"]
        assert np.array_equal(bits(xt.cpu().numpy()), bits(xt_ref))
        zl2, zu2 = dv["zl"].clone(), dv["zu"].clone()
        zl2[::3] *= 1e12
        zu2[1::3] *= 1e-14
        ozl, ozu = zl2.cpu().numpy().copy(), zu2.cpu().numpy().copy()
        nl.clip_duals(xt.data_ptr(), mu, zl2.data_ptr(), zu2.data_ptr())
        nl.sync()
        L.orc_clip_duals(n, O._dp_(O.f64(xt_ref)), O._dp_(O.f64(inst.lb)), O._dp_(O.f64(inst.ub)), mu,
                         O._dp_(ozl), O._dp_(ozu))
        assert np.array_equal(bits(zl2.cpu().numpy()), bits(ozl))
        assert np.array_equal(bits(zu2.cpu().numpy()), bits(ozu))
        # outer update of y_k (solver.cpp:213-217)
        yk = dv["yk"].clone()
        rn = nl.outer(dv["r"].data_ptr(), yk.data_ptr(), rho, 1)
        nl.sync()
        assert rn == np.abs(st["r"]).max()
        assert np.array_equal(bits(yk.cpu().numpy()), bits(st["yk"] + rho * st["r"]))
