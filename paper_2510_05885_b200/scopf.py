"""Security-constrained OPF with N-1 contingency blocks, sharded over GPUs.

SURVEY.md 8(d) config #5 / 8(e).  The reference has no SCOPF instance (the
paper's SCOPF, comes from an external model); this is the
repo's generator of the same *structure*: a base network plus K blocks (block
0 the intact network, block k >= 1 with branch (k-1) mod n_e out), coupled
only through the base generator set-points p0 (preventive dispatch with a
penalised per-block recourse r^k):

    min  sum_i w_i (p0_i - pref_i)^2 + sum_k sum_i c_r (r^k_i)^2
    s.t. p0_i + r^k_i - d_i - sum_{e in E_k at i} (+-) b_e sin(th^k_a - th^k_b) = 0
         -0.8 b_e <= b_e sin(th^k_a - th^k_b) <= 0.8 b_e        (e in E_k)
         0 <= p0 <= 10, -0.5 <= r^k <= 0.5, -1 <= th^k <= 1, th^k_0 = 0

in the reference's NLP conventions (Jacobian CSR with sorted columns,
equality rows first, one slack per inequality row appended after t, Hessian
lower CSC = grad^2 f - sum y grad^2 c; the same per-bus model as
proj/src/problems.cpp:342-414).  Variable order t = [p0 | th^0 r^0 | th^1 r^1
| ...]; rows eq = [balance of block 0 | block 1 | ...], ineq = [flows of
block 0 | ...].

The condensed KKT matrix (K1s, N = nt) is block-arrowhead: blocks couple only
through p0.  ``subproblem`` gives rank g the blocks [k0, k1) with p0 in
front; the ranks' K1s matrices sum to the global one (K is additive over
constraint rows and Hessian terms) once the p0 terms that must count once --
the objective Hessian, sigma and rbar1 of p0, and delta on p0's diagonal --
are kept on the owner only (delta is corrected after the sum).
``ScopfKkt`` is the distributed ``KktContext::solve`` (kkt.cpp:266-314) on
those shares: each GPU factors its blocks in Schur mode (ncl_schur_*), the
n0 x n0 Schur complement, the reduced right-hand sides and the inertia /
perturbed counts are summed with torch.distributed (NCCL over NVLink), and
every rank factors and solves the dense Schur system redundantly (Haynsworth:
inertia(K) = sum_k inertia(A_kk) + inertia(S), so the delta loop decides
identically everywhere).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .instances import MT19937_64, Instance, _csr_from_rows, _lower_csc_from_pairs, ring_chord_edges

C_R = 10.0           # recourse penalty
FLOW_FRAC = 0.8      # flow limit as a fraction of the susceptance


@dataclass
class ScopfData:
    nbus: int
    K: int
    seed: int
    edges: np.ndarray
    susc: np.ndarray
    pref: np.ndarray
    weight: np.ndarray
    demand: np.ndarray


def scopf_data(nbus: int, K: int, seed: int) -> ScopfData:
    """network data from the reference RNG (problems.cpp:17-24 semantics),
    ring-with-chords topology (problems.cpp:346-349)"""
    edges = np.asarray(ring_chord_edges(nbus), np.int64).reshape(-1, 2)
    ne = len(edges)
    rng = MT19937_64(seed)
    susc = rng.uniform(1.0, 3.0, ne)
    theta_ref = np.zeros(nbus)
    theta_ref[1:] = rng.uniform(-0.3, 0.3, nbus - 1)
    pref = rng.uniform(1.0, 2.0, nbus)
    weight = rng.uniform(0.5, 2.0, nbus)
    demand = pref.copy()
    for e in range(ne):
        i, j = edges[e]
        f = susc[e] * np.sin(theta_ref[i] - theta_ref[j])
        demand[i] -= f
        demand[j] += f
    return ScopfData(nbus, K, seed, edges, susc, pref, weight, demand)


def block_edges(D: ScopfData, k: int) -> np.ndarray:
    """edge ids present in block k (block 0 intact, block k drops k-1 mod ne)"""
    ne = len(D.edges)
    ids = np.arange(ne)
    return ids if k == 0 else np.delete(ids, (k - 1) % ne)


class ScopfInstance(Instance):
    pass


def subproblem(D: ScopfData, k0: int, k1: int, owner: bool) -> Instance:
    """NLP of blocks [k0, k1) with the coupling set-points p0 first.
    (0, K, True) is the global problem."""
    nb = D.nbus
    n0 = nb
    nbk = k1 - k0
    nt = n0 + nbk * 2 * nb
    eq_rows, in_rows, pairs = [], [], []
    lb_s, ub_s = [], []
    pairs.append(np.stack([np.arange(n0), np.arange(n0)], 1))  # p0 objective (pattern on every rank)
    blk = []  # per block: (vo, edge ids, ineq row offset, eq row offset)
    n_in = 0
    for kk, k in enumerate(range(k0, k1)):
        vo = n0 + kk * 2 * nb
        eids = block_edges(D, k)
        E = D.edges[eids]
        a, b = E[:, 0], E[:, 1]
        inc = [set() for _ in range(nb)]
        for i, j in E:
            inc[i].update((int(i), int(j)))
            inc[j].update((int(i), int(j)))
        for i in range(nb):
            eq_rows.append([i] + [vo + j for j in sorted(inc[i])] + [vo + nb + i])
        for i, j in E:
            in_rows.append(sorted((vo + int(i), vo + int(j))))
        pairs.append(np.stack([vo + a, vo + a], 1))
        pairs.append(np.stack([vo + b, vo + b], 1))
        pairs.append(np.stack([vo + np.maximum(a, b), vo + np.minimum(a, b)], 1))
        pairs.append(np.stack([vo + nb + np.arange(nb)] * 2, 1))
        lb_s.append(-FLOW_FRAC * D.susc[eids])
        ub_s.append(FLOW_FRAC * D.susc[eids])
        blk.append((k, vo, eids, n_in))
        n_in += len(eids)
    m_eq = len(eq_rows)
    jp_ptr, jp_idx = _csr_from_rows(eq_rows + in_rows)
    hp_ptr, hp_idx = _lower_csc_from_pairs(nt, np.concatenate(pairs))
    lb = np.full(nt, -1.0)
    ub = np.full(nt, 1.0)
    lb[:n0], ub[:n0] = 0.0, 10.0
    for k, vo, _, _ in blk:
        lb[vo] = ub[vo] = 0.0                     # reference angle of block k
        lb[vo + nb:vo + 2 * nb], ub[vo + nb:vo + 2 * nb] = -0.5, 0.5
    lb = np.concatenate([lb] + lb_s)
    ub = np.concatenate([ub] + ub_s)
    start = np.zeros(nt)
    start[:n0] = 1.5
    inst = Instance(f"scopf:{nb}:{D.K}:{D.seed}[{k0}:{k1}]", nt, n_in, m_eq, m_eq + n_in,
                    hp_ptr, hp_idx, jp_ptr, jp_idx, lb, ub, start)
    inst.scopf = dict(data=D, k0=k0, k1=k1, owner=owner, n0=n0, blocks=blk)
    return inst


def _slots(ptr, idx, rows, cols):
    """position of (row r, col c) in a CSR/CSC given as (ptr over rows, idx = cols)"""
    out = np.empty(len(rows), np.int64)
    for q in range(len(rows)):
        r0, r1 = ptr[rows[q]], ptr[rows[q] + 1]
        out[q] = r0 + np.searchsorted(idx[r0:r1], cols[q])
    return out


def scopf_case(inst: Instance, seed: int, rho: float = 100.0):
    """KktInput of a (sub)problem in the test_kkt.cpp:40-68 recipe, drawn per
    block (seed, block) so that every rank's share is the matching slice of
    the global case: t = start + U(-.05,.05), y ~ U(-.01,.01) -> hval, jval;
    sigma ~ U(.5,2), rbar1 ~ U(-1,1), rbar2, rbar3 ~ U(-1,1).  p0's sigma,
    rbar1 and objective Hessian live on the owner only (zero elsewhere)."""
    S = inst.scopf
    D, n0, nb = S["data"], S["n0"], S["data"].nbus
    nt, m_eq = inst.nt, inst.m_eq
    hval = np.zeros(len(inst.hp_idx))
    jval = np.zeros(len(inst.jp_idx))
    sigma = np.zeros(inst.n)
    rbar1 = np.zeros(inst.n)
    rbar2 = np.zeros(inst.m)
    rbar3 = np.zeros(inst.m)
    r0 = MT19937_64(seed * 1000003 + 7)
    t0 = 1.5 + r0.uniform(-0.05, 0.05, n0)
    s0, q0 = r0.uniform(0.5, 2.0, n0), r0.uniform(-1.0, 1.0, n0)
    hp_ptr, hp_idx, jp_ptr, jp_idx = inst.hp_ptr, inst.hp_idx, inst.jp_ptr, inst.jp_idx
    # H lower CSC: column c holds rows >= c; a diagonal (i, i) slot
    diag = lambda cols: _slots(hp_ptr, hp_idx, cols, cols)
    if S["owner"]:
        hval[diag(np.arange(n0))] = 2.0 * D.weight
        sigma[:n0], rbar1[:n0] = s0, q0
    for kk, (k, vo, eids, io) in enumerate(S["blocks"]):
        rb = MT19937_64(seed * 1000003 + 11 + k)
        ne_k = len(eids)
        tk = rb.uniform(-0.05, 0.05, 2 * nb)        # start of th, r is 0
        yk = rb.uniform(-0.01, 0.01, nb + ne_k)
        th, rr = tk[:nb], tk[nb:]
        E = D.edges[eids]
        a, b = E[:, 0], E[:, 1]
        dth = th[a] - th[b]
        sn = D.susc[eids] * np.sin(dth)
        cs = D.susc[eids] * np.cos(dth)
        ybal, yflow = yk[:nb], yk[nb:]
        # Jacobian: balance rows kk*nb + i, flow rows m_eq + io + e
        brow = kk * nb
        jval[_slots(jp_ptr, jp_idx, brow + np.arange(nb), np.arange(nb))] += 1.0
        jval[_slots(jp_ptr, jp_idx, brow + np.arange(nb), vo + nb + np.arange(nb))] += 1.0
        np.add.at(jval, _slots(jp_ptr, jp_idx, brow + a, vo + a), -cs)
        np.add.at(jval, _slots(jp_ptr, jp_idx, brow + a, vo + b), cs)
        np.add.at(jval, _slots(jp_ptr, jp_idx, brow + b, vo + a), cs)
        np.add.at(jval, _slots(jp_ptr, jp_idx, brow + b, vo + b), -cs)
        frow = m_eq + io + np.arange(ne_k)
        jval[_slots(jp_ptr, jp_idx, frow, vo + a)] += cs
        jval[_slots(jp_ptr, jp_idx, frow, vo + b)] += -cs
        # Hessian: recourse objective + constraint curvature (-y grad^2 c)
        hval[diag(vo + nb + np.arange(nb))] += 2.0 * C_R
        coef = ybal[a] - ybal[b] - yflow
        np.add.at(hval, diag(vo + a), coef * (-sn))
        np.add.at(hval, diag(vo + b), coef * (-sn))
        hi, lo = vo + np.maximum(a, b), vo + np.minimum(a, b)
        np.add.at(hval, _slots(hp_ptr, hp_idx, lo, hi), coef * sn)
        # sigma / rbar over block variables and slacks; rbar2/3 over rows
        sv = rb.uniform(0.5, 2.0, 2 * nb + ne_k)
        qv = rb.uniform(-1.0, 1.0, 2 * nb + ne_k)
        sigma[vo:vo + 2 * nb], sigma[nt + io:nt + io + ne_k] = sv[:2 * nb], sv[2 * nb:]
        rbar1[vo:vo + 2 * nb], rbar1[nt + io:nt + io + ne_k] = qv[:2 * nb], qv[2 * nb:]
        r2 = rb.uniform(-1.0, 1.0, nb + ne_k)
        r3 = rb.uniform(-1.0, 1.0, nb + ne_k)
        rbar2[brow:brow + nb], rbar2[frow] = r2[:nb], r2[nb:]
        rbar3[brow:brow + nb], rbar3[frow] = r3[:nb], r3[nb:]
    _ = t0  # p0 enters the model linearly: its values do not reach hval/jval
    return dict(hval=hval, jval=jval, sigma=sigma, rbar1=rbar1, rbar2=rbar2, rbar3=rbar3, rho=rho)


def block_range(K: int, world: int, rank: int):
    """contiguous block shares, ceil(K / world) each"""
    per = (K + world - 1) // world
    return min(K, rank * per), min(K, (rank + 1) * per)


def global_maps(D: ScopfData, sub: Instance, glob: Instance):
    """index maps of a rank's share into the global problem: local t-variable
    -> global t-variable, local slack -> global slack, local row -> global row"""
    S = sub.scopf
    nb, n0 = D.nbus, S["n0"]
    tv = [np.arange(n0)]
    sv, er, ir = [], [], []
    gio = {}
    acc = 0
    for k in range(D.K):
        gio[k] = acc
        acc += len(block_edges(D, k))
    for kk, (k, vo, eids, io) in enumerate(S["blocks"]):
        tv.append(n0 + k * 2 * nb + np.arange(2 * nb))
        sv.append(gio[k] + np.arange(len(eids)))
        er.append(k * nb + np.arange(nb))
        ir.append(glob.m_eq + gio[k] + np.arange(len(eids)))
    tmap = np.concatenate(tv)
    smap = np.concatenate(sv) if sv else np.zeros(0, np.int64)
    rmap = np.concatenate(er + ir) if er else np.zeros(0, np.int64)
    return tmap, smap, rmap


def parse_spec(spec: str):
    """'scopf:<nbus>:<K>:<seed>'"""
    t = spec.split(":")
    if t[0] != "scopf" or len(t) != 4:
        raise ValueError(f"bad scopf spec {spec}")
    return int(t[1]), int(t[2]), int(t[3])


# ---------------------------------------------------------------------------
class ScopfKkt:
    """Distributed ``KktContext::solve`` (kkt.cpp:266-314, K1s) of a SCOPF over
    the ranks of the default process group (or a single process).

    Every rank owns a ``subproblem`` share in Schur mode on its GPU.  Per
    factorization attempt: local refill + block factorization -> S_g;
    all_reduce(S) and all_reduce(n_pos, n_neg, perturbed, fail); every rank
    factors S.  Per solve: forward through the blocks -> reduced rhs;
    all_reduce; dense solve; backward.  Refinement (sparse.cpp:278-322) and
    the acceptance test use global norms (max all_reduce).  Inputs / outputs
    are this rank's slices (torch float64 CUDA tensors)."""

    def __init__(self, sub: Instance, nt_global: int, opts=None, dist=None):
        import ctypes as C

        import torch

        from . import _lib
        from ._lib import check, ip

        self.torch = torch
        self.dist = dist
        self.world = dist.get_world_size() if dist is not None else 1
        self.rank = dist.get_rank() if dist is not None else 0
        _lib.require_gpu()
        self.L = _lib.lib()
        self.sub = sub
        self.n0 = sub.scopf["n0"]
        self.nt_global = nt_global
        o = opts or (1e-10, 10, 1e-12, 1e40, 1e-8)
        self.opts = _lib.KktOpts(*o)
        keep = [np.ascontiguousarray(a, np.int32) for a in (sub.hp_ptr, sub.hp_idx, sub.jp_ptr, sub.jp_idx)]
        h = C.c_void_p()
        check(self.L.ncl_schur_create(sub.nt, ip(keep[0]), ip(keep[1]), sub.m, ip(keep[2]), ip(keep[3]),
                                      sub.ns, sub.m_eq, self.n0, C.byref(self.opts), C.byref(h)),
              "ncl_schur_create")
        self.h = h
        self._check = check
        dev = torch.device("cuda")
        f64 = dict(dtype=torch.float64, device=dev)
        self.N = sub.nt
        self.S = torch.zeros(self.n0, self.n0, **f64)
        self.b = torch.zeros(self.N, **f64)
        self.b0 = torch.zeros(self.n0, **f64)
        self.x0 = torch.zeros(self.n0, **f64)
        self.bufs = {k: torch.zeros(self.N, **f64) for k in ("x", "r", "dx", "xn", "rn", "rr")}
        self.stats = (C.c_int * 4)()
        self.C = C

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ncl_schur_destroy(self.h)
            self.h = None

    # -- collectives ---------------------------------------------------------
    def _sum(self, t):
        if self.dist is not None and self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t

    def _max(self, v: float) -> float:
        if self.dist is None or self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def _p(self, t):
        return self.C.c_void_p(t.data_ptr())

    # -- distributed pieces ---------------------------------------------------
    def _factor(self, hv, jv, sg, rho, delta):
        torch = self.torch
        torch.cuda.synchronize()
        self._check(self.L.ncl_schur_factor(self.h, self._p(hv), self._p(jv), self._p(sg), rho, delta,
                                            self.stats, self._p(self.S)), "ncl_schur_factor")
        loc = torch.tensor(list(self.stats), dtype=torch.float64, device="cuda")
        self._sum(self.S)
        self._sum(loc)
        torch.cuda.synchronize()
        # delta reached p0's diagonal once per rank: keep one
        self._check(self.L.ncl_schur_factor_dense(self.h, self._p(self.S), -(self.world - 1) * delta,
                                                  self.stats), "ncl_schur_factor_dense")
        g = [int(v) for v in loc.tolist()]
        n_pos, n_neg, pert = g[0] + self.stats[0], g[1] + self.stats[1], g[2] + self.stats[2]
        ok = g[3] == 0 and self.stats[3] == 0
        return ok, n_pos, n_neg, pert

    def _solve(self, b, x):
        """x = K^-1 b; b's p0 part is this rank's partial sum"""
        torch = self.torch
        torch.cuda.synchronize()
        self._check(self.L.ncl_schur_forward(self.h, self._p(b), self._p(self.b0)), "ncl_schur_forward")
        self._sum(self.b0)
        torch.cuda.synchronize()
        self._check(self.L.ncl_schur_solve0(self.h, self._p(self.b0), self._p(self.x0)), "ncl_schur_solve0")
        self._check(self.L.ncl_schur_backward(self.h, self._p(self.x0), self._p(x)), "ncl_schur_backward")

    def _residual(self, x, b, r, delta):
        """r = b - K x (global rows of this rank: p0 part summed and identical
        on every rank); returns ||r||_inf over the whole system"""
        torch = self.torch
        torch.cuda.synchronize()
        self._check(self.L.ncl_schur_residual(self.h, self._p(x), self._p(b), self._p(r)), "ncl_schur_residual")
        r0 = r[:self.n0]
        self._sum(r0)
        r0 += (self.world - 1) * delta * x[:self.n0]
        loc = float(r[self.n0:].abs().max().item()) if self.N > self.n0 else 0.0
        return self._max(max(loc, float(r0.abs().max().item())))

    def _owner_part(self, v):
        """a globally summed p0 vector enters a solve from the owner only"""
        if self.rank != 0:
            v[:self.n0] = 0.0
        return v

    def _solve_refined(self, b, delta):
        """sparse.cpp:278-322 on the distributed system"""
        o = self.opts
        B = self.bufs
        x = B["x"]
        self._solve(b, x)
        b0 = b[:self.n0].clone()
        self._sum(b0)
        loc = float(b[self.n0:].abs().max().item()) if self.N > self.n0 else 0.0
        bn = self._max(max(loc, float(b0.abs().max().item())))
        bfull = b.clone()
        bfull[:self.n0] = b0                       # the summed rhs, for residuals
        bres = self._owner_part(bfull.clone())      # residual input: p0 rhs once
        r = B["r"]
        res = self._residual(x, bres, r, delta)
        denom = bn if bn > 0.0 else 1.0
        prev, stagnant, steps = res, 0, 0
        while steps < o.max_refine and res > o.refine_tol * denom:
            rr = B["rr"]
            rr.copy_(r)
            self._owner_part(rr)
            dx = B["dx"]
            self._solve(rr, dx)
            xn = B["xn"]
            torch = self.torch
            torch.add(x, dx, out=xn)
            rn = B["rn"]
            res_new = self._residual(xn, bres, rn, delta)
            if not np.isfinite(res_new) or res_new >= res:
                break
            x.copy_(xn)
            r.copy_(rn)
            steps += 1
            stagnant = stagnant + 1 if res_new > 0.5 * prev else 0
            prev = res = res_new
            if stagnant >= 2:
                break
        return x, steps, res / denom, bn, res

    def solve(self, case, rho: float, warm: float = 0.0):
        """case: dict of this rank's torch tensors (hval, jval, sigma, rbar1,
        rbar2, rbar3).  Returns a dict like KktStep (kkt.hpp:48-56)."""
        torch = self.torch
        hv, jv, sg = case["hval"], case["jval"], case["sigma"]
        o = self.opts
        hmax = self._max(max(float(hv.abs().max().item()) if hv.numel() else 0.0,
                             float(sg.abs().max().item()) if sg.numel() else 0.0))
        delta, first, attempts = 0.0, True, 0
        dx = torch.zeros(self.sub.n, dtype=torch.float64, device="cuda")
        dr = torch.zeros(self.sub.m, dtype=torch.float64, device="cuda")
        dy = torch.zeros(self.sub.m, dtype=torch.float64, device="cuda")
        while True:
            attempts += 1
            ok, n_pos, n_neg, pert = self._factor(hv, jv, sg, rho, delta)
            if ok and n_pos == self.nt_global and n_neg == 0:
                torch.cuda.synchronize()
                self._check(self.L.ncl_schur_rhs(self.h, self._p(jv), self._p(sg), self._p(case["rbar1"]),
                                                 self._p(case["rbar2"]), self._p(case["rbar3"]), rho, delta,
                                                 self._p(self.b)), "ncl_schur_rhs")
                x, steps, rel, bn, res = self._solve_refined(self.b, delta)
                if pert == 0 or res <= o.accept_tol * max(1.0, bn):
                    torch.cuda.synchronize()
                    self._check(self.L.ncl_schur_recover(self.h, self._p(jv), self._p(x), self._p(case["rbar2"]),
                                                         rho, delta, self._p(dx), self._p(dr), self._p(dy)),
                                "ncl_schur_recover")
                    fin = all(bool(torch.isfinite(v).all()) for v in (dx, dr, dy))
                    fin = self._max(0.0 if fin else 1.0) == 0.0
                    return dict(dx=dx, dr=dr, dy=dy, delta=delta, factor_attempts=attempts,
                                refine_steps=steps, perturbed_pivots=pert, rel_residual=rel, ok=fin)
            if first:
                delta = max(1e-20, warm / 3.0) if warm > 0.0 else 1e-8 * max(1.0, hmax)
                first = False
            else:
                delta *= 8.0
            if delta > o.delta_max:
                return dict(dx=dx, dr=dr, dy=dy, delta=delta, factor_attempts=attempts, refine_steps=0,
                            perturbed_pivots=0, rel_residual=0.0, ok=False)
