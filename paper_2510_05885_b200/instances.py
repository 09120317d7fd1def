"""Synthetic KKT inputs of the reference's instance families (numpy).

The reference builds its problems through the ExprGraph API and differentiates
them with its own AD (proj/src/problems.cpp, proj/src/model.cpp).  The GPU
benchmark needs the same *shapes* at sizes the registry does not have, on a
box where the reference does not exist, so the families are restated here
with analytic derivatives:

* ``opf_graph`` -- proj/src/problems.cpp:342-414 on any edge list: the ring
  with chords (``opf_toy``) and a 4-neighbour grid (``opf_mesh``, the bushier
  perf variant of SURVEY.md section 8(d)).  Data generation consumes the
  reference RNG (problems.cpp:17-24, std::mt19937_64) in the reference order,
  so ``opf_toy(500, 203)`` is the registry's ``opf-toy-1000``.
* ``mpcc_sep`` -- problems.cpp:287-305.

Patterns follow the reference's Model conventions exactly (Jacobian CSR rows
eq-then-ineq with sorted columns; Hessian lower CSC as the sorted union of
nonlinear-element variable pairs, model.cpp:154-186); tests/test_instances.py
checks them against the reference Model bit for bit and the values to
rounding.  ``kkt_case`` is the test_kkt.cpp:40-68 recipe.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (Matsumoto & Nishimura 64-bit MT), vectorised twist."""
    NN, MM = 312, 156
    A = np.uint64(0xB5026F5AA96619E9)
    UM = np.uint64(0xFFFFFFFF80000000)
    LM = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [0] * self.NN
        mt[0] = seed & _M64
        for i in range(1, self.NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt = np.array(mt, dtype=np.uint64)
        self.buf = np.zeros(0, dtype=np.uint64)
        self.pos = 0

    def _twist(self):
        mt = self.mt
        NN, MM = self.NN, self.MM
        one = np.uint64(1)
        zero = np.uint64(0)

        def step(i0, i1, src_m):
            x = (mt[i0:i1] & self.UM) | (mt[i0 + 1:i1 + 1] & self.LM)
            mag = np.where((x & one) == one, self.A, zero)
            mt[i0:i1] = src_m ^ (x >> one) ^ mag

        step(0, NN - MM, mt[MM:NN].copy())
        step(NN - MM, NN - 1, mt[0:MM - 1].copy())
        x = (mt[NN - 1] & self.UM) | (mt[0] & self.LM)
        mag = self.A if int(x) & 1 else zero
        mt[NN - 1] = mt[MM - 1] ^ (x >> one) ^ mag
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self.buf = y
        self.pos = 0

    def raw(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        k = 0
        while k < n:
            if self.pos >= len(self.buf):
                self._twist()
            take = min(n - k, len(self.buf) - self.pos)
            out[k:k + take] = self.buf[self.pos:self.pos + take]
            self.pos += take
            k += take
        return out

    def uniform(self, lo: float, hi: float, n: int) -> np.ndarray:
        """lo + (hi - lo) * ((g >> 11) * 2^-53), problems.cpp:20-23"""
        u = (self.raw(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        return lo + (hi - lo) * u


@dataclass
class Instance:
    name: str
    nt: int
    ns: int
    m_eq: int
    m: int
    hp_ptr: np.ndarray
    hp_idx: np.ndarray
    jp_ptr: np.ndarray
    jp_idx: np.ndarray
    lb: np.ndarray      # NLP-form bounds, length n = nt + ns
    ub: np.ndarray
    start: np.ndarray   # length nt
    evaluator: object = None

    @property
    def n(self) -> int:
        return self.nt + self.ns


def _csr_from_rows(rows):
    ptr = np.zeros(len(rows) + 1, np.int32)
    for i, r in enumerate(rows):
        ptr[i + 1] = ptr[i] + len(r)
    idx = np.concatenate([np.asarray(r, np.int32) for r in rows]) if rows else np.zeros(0, np.int32)
    return ptr, idx.astype(np.int32)


def _lower_csc_from_pairs(n, pairs):
    """pairs: array (k, 2) of (row i >= col j); sorted unique by (col, row)."""
    if len(pairs) == 0:
        return np.zeros(n + 1, np.int32), np.zeros(0, np.int32)
    p = np.unique(pairs[:, 1].astype(np.int64) * (1 << 32) + pairs[:, 0].astype(np.int64))
    col = (p >> 32).astype(np.int32)
    row = (p & 0xffffffff).astype(np.int32)
    ptr = np.zeros(n + 1, np.int32)
    np.add.at(ptr, col + 1, 1)
    return np.cumsum(ptr).astype(np.int32), row


def _slot_index(hp_ptr, hp_idx, rows, cols):
    """positions of (row, col) entries in the lower CSC (vectorised)."""
    n = len(hp_ptr) - 1
    key = cols.astype(np.int64) * (n + 1) + rows.astype(np.int64)
    colv = np.repeat(np.arange(n, dtype=np.int64), np.diff(hp_ptr))
    allkey = colv * (n + 1) + hp_idx.astype(np.int64)
    pos = np.searchsorted(allkey, key)
    assert np.all(allkey[pos] == key)
    return pos


class _OpfEval:
    def __init__(self, nbus, edges, susc, weight, inj_ref, demand, inst):
        self.nbus, self.edges, self.susc = nbus, edges, susc
        self.weight, self.inj_ref, self.demand = weight, inj_ref, demand
        self.inst = inst
        nb = nbus
        a, b = edges[:, 0], edges[:, 1]
        ne = len(edges)
        # Jacobian slot positions of each edge contribution
        jp_ptr, jp_idx = inst.jp_ptr, inst.jp_idx

        def pos_in_row(rows, cols):
            out = np.empty(len(rows), np.int64)
            for k in range(len(rows)):
                r0, r1 = jp_ptr[rows[k]], jp_ptr[rows[k] + 1]
                out[k] = r0 + np.searchsorted(jp_idx[r0:r1], cols[k])
            return out

        self.j_bal_inj = pos_in_row(np.arange(nb), nb + np.arange(nb))
        self.j_bal_a_a = pos_in_row(a, a)   # row a (from) wrt theta_a
        self.j_bal_a_b = pos_in_row(a, b)
        self.j_bal_b_a = pos_in_row(b, a)
        self.j_bal_b_b = pos_in_row(b, b)
        self.j_flow_a = pos_in_row(nb + np.arange(ne), a)
        self.j_flow_b = pos_in_row(nb + np.arange(ne), b)
        hp_ptr, hp_idx = inst.hp_ptr, inst.hp_idx
        self.h_aa = _slot_index(hp_ptr, hp_idx, a, a)
        self.h_bb = _slot_index(hp_ptr, hp_idx, b, b)
        self.h_ab = _slot_index(hp_ptr, hp_idx, np.maximum(a, b), np.minimum(a, b))
        self.h_inj = _slot_index(hp_ptr, hp_idx, nb + np.arange(nb), nb + np.arange(nb))

    def eval(self, t, y):
        """hval (obj_scale 1, multipliers y), jval, grad (nt), c (m)."""
        nb = self.nbus
        a, b = self.edges[:, 0], self.edges[:, 1]
        ne = len(a)
        th = t[:nb]
        inj = t[nb:]
        dth = th[a] - th[b]
        sn = self.susc * np.sin(dth)
        cs = self.susc * np.cos(dth)
        inst = self.inst
        jval = np.zeros(len(inst.jp_idx))
        np.add.at(jval, self.j_bal_inj, 1.0)
        # row a: -f_e ; row b: +f_e
        np.add.at(jval, self.j_bal_a_a, -cs)
        np.add.at(jval, self.j_bal_a_b, cs)
        np.add.at(jval, self.j_bal_b_a, cs)
        np.add.at(jval, self.j_bal_b_b, -cs)
        jval[self.j_flow_a] += cs
        jval[self.j_flow_b] += -cs
        # Hessian: obj 2 w_i on inj; constraints -y_i * d2 c_i
        hval = np.zeros(len(inst.hp_idx))
        hval[self.h_inj] += 2.0 * self.weight
        ya, yb, yf = y[a], y[b], y[nb:nb + ne]
        # d2 f_e: (aa) -s, (bb) -s, (ab) +s with s = susc sin
        coef = -ya * (-1.0) + -yb * (1.0) + -yf  # multiplier of d2 f_e
        np.add.at(hval, self.h_aa, coef * (-sn))
        np.add.at(hval, self.h_bb, coef * (-sn))
        np.add.at(hval, self.h_ab, coef * sn)
        grad = np.zeros(inst.nt)
        grad[nb:] = 2.0 * self.weight * (inj - self.inj_ref)
        c = np.zeros(inst.m)
        bal = inj - self.demand
        np.add.at(bal, a, -sn)
        np.add.at(bal, b, sn)
        c[:nb] = bal
        c[nb:] = sn
        return hval, jval, grad, c


def opf_graph(name: str, nbus: int, edges, seed: int) -> Instance:
    """proj/src/problems.cpp:342-414 on an arbitrary edge list."""
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    ne = len(edges)
    rng = MT19937_64(seed)
    susc = rng.uniform(1.0, 3.0, ne)
    theta_ref = np.zeros(nbus)
    theta_ref[1:] = rng.uniform(-0.3, 0.3, nbus - 1)
    inj_ref = rng.uniform(1.0, 2.0, nbus)
    weight = rng.uniform(0.5, 2.0, nbus)
    demand = inj_ref.copy()
    for e in range(ne):  # sequential accumulation order of the reference
        i, j = edges[e]
        f = susc[e] * np.sin(theta_ref[i] - theta_ref[j])
        demand[i] -= f
        demand[j] += f
    nt = 2 * nbus
    # Jacobian rows: balance (theta of incident edge ends + own injection),
    # then one row per edge flow
    inc = [set() for _ in range(nbus)]
    for i, j in edges:
        inc[i].update((int(i), int(j)))
        inc[j].update((int(i), int(j)))
    rows = [sorted(inc[i]) + [nbus + i] for i in range(nbus)]
    rows += [sorted((int(i), int(j))) for i, j in edges]
    jp_ptr, jp_idx = _csr_from_rows(rows)
    a, b = edges[:, 0], edges[:, 1]
    pairs = np.concatenate([
        np.stack([a, a], 1), np.stack([b, b], 1), np.stack([np.maximum(a, b), np.minimum(a, b)], 1),
        np.stack([nbus + np.arange(nbus)] * 2, 1)])
    hp_ptr, hp_idx = _lower_csc_from_pairs(nt, pairs)
    ns = ne
    lb = np.concatenate([np.full(nt, -1.0), -0.8 * susc])
    ub = np.concatenate([np.full(nt, 1.0), 0.8 * susc])
    lb[0] = ub[0] = 0.0
    lb[nbus:nt] = 0.0
    ub[nbus:nt] = 10.0
    start = np.zeros(nt)
    start[nbus:] = 1.5
    inst = Instance(name, nt, ns, nbus, nbus + ne, hp_ptr, hp_idx, jp_ptr, jp_idx, lb, ub, start)
    inst.evaluator = _OpfEval(nbus, edges, susc, weight, inj_ref, demand, inst)
    return inst


def ring_chord_edges(nbus: int):
    """problems.cpp:346-349"""
    e = [(i, (i + 1) % nbus) for i in range(nbus)]
    if nbus > 10:
        e += [(i, (i + 3) % nbus) for i in range(0, nbus, 5)]
    return e


def mesh_edges(nx: int, ny: int):
    e = []
    for r in range(ny):
        for c in range(nx):
            bsn = r * nx + c
            if c + 1 < nx:
                e.append((bsn, bsn + 1))
            if r + 1 < ny:
                e.append((bsn, bsn + nx))
    return e


def opf_toy(nbus: int, seed: int) -> Instance:
    return opf_graph(f"opf_toy:{nbus}:{seed}", nbus, ring_chord_edges(nbus), seed)


def opf_mesh(nx: int, ny: int, seed: int) -> Instance:
    return opf_graph(f"opf_mesh:{nx}:{ny}:{seed}", nx * ny, mesh_edges(nx, ny), seed)


class _MpccEval:
    def __init__(self, pairs, inst):
        self.P = pairs
        self.inst = inst

    def eval(self, t, y):
        P = self.P
        a, c = t[0::2], t[1::2]
        jval = np.empty(2 * P)
        jval[0::2] = c
        jval[1::2] = a
        hval = np.empty(3 * P)  # per pair: (a,a), (c,a), (c,c) in CSC order
        hval[0::3] = 2.0
        hval[1::3] = -y
        hval[2::3] = 2.0
        grad = np.empty(2 * P)
        grad[0::2] = 2.0 * (a - 1.0)
        grad[1::2] = 2.0 * (c - 1.0)
        return hval, jval, grad, a * c


def mpcc_sep(pairs: int) -> Instance:
    """problems.cpp:287-305"""
    nt = 2 * pairs
    jp_ptr = (2 * np.arange(pairs + 1)).astype(np.int32)
    jp_idx = np.arange(nt, dtype=np.int32)
    hp_ptr = np.zeros(nt + 1, np.int32)
    hp_ptr[1::2] = 0
    cnt = np.tile([2, 1], pairs)
    hp_ptr[1:] = np.cumsum(cnt)
    hp_idx = np.empty(3 * pairs, np.int32)
    hp_idx[0::3] = 2 * np.arange(pairs)
    hp_idx[1::3] = 2 * np.arange(pairs) + 1
    hp_idx[2::3] = 2 * np.arange(pairs) + 1
    lb = np.zeros(nt)
    ub = np.full(nt, np.inf)
    inst = Instance(f"mpcc_sep:{pairs}", nt, 0, pairs, pairs, hp_ptr, hp_idx, jp_ptr, jp_idx, lb, ub,
                    np.full(nt, 0.5))
    inst.evaluator = _MpccEval(pairs, inst)
    return inst


class _ElecEval:
    """COPS 'elec' (integration/instances.hpp elec): Coulomb potential of np
    points, sum_{i<j} 1 / |p_i - p_j|, constraints |p_i|^2 - 1 = 0.  The
    Hessian pattern is the dense lower triangle (every pair of points shares
    a nonlinear element)."""

    def __init__(self, npt, inst):
        self.np = npt
        self.inst = inst
        n = 3 * npt
        c = np.arange(n, dtype=np.int64)
        self.colstart = c * n - c * (c - 1) // 2  # slot of (c, c) in the dense lower CSC

    def eval(self, t, y):
        npt, n = self.np, 3 * self.np
        P = t.reshape(npt, 3)
        H = np.zeros((n, n))
        grad = np.zeros(n)
        for i in range(npt):
            d = P[i] - P            # (np, 3)
            r2 = (d * d).sum(1)
            r2[i] = 1.0
            r = np.sqrt(r2)
            inv3, inv5 = 1.0 / (r2 * r), 1.0 / (r2 * r2 * r)
            B = 3.0 * d[:, :, None] * d[:, None, :] * inv5[:, None, None] - \
                np.eye(3)[None] * inv3[:, None, None]
            B[i] = 0.0
            H[3 * i:3 * i + 3, 3 * i:3 * i + 3] += B.sum(0)
            H[3 * i:3 * i + 3, :] -= B.transpose(1, 0, 2).reshape(3, n)
            g = -d * inv3[:, None]
            g[i] = 0.0
            grad[3 * i:3 * i + 3] = g.sum(0)
        for i in range(npt):  # -y_i * grad^2 (|p_i|^2 - 1) = -2 y_i I
            H[3 * i + np.arange(3), 3 * i + np.arange(3)] += -2.0 * y[i]
        hval = np.concatenate([H[c:, c] for c in range(n)])
        jval = (2.0 * P).reshape(-1)
        cval = (P * P).sum(1) - 1.0
        return hval, jval, grad, cval


def elec(npt: int, seed: int) -> Instance:
    """integration/instances.hpp elec (COPS 3.0): seeded start on the sphere
    (problems.cpp:17-24 Rng draws th, ph per point in order)."""
    n = 3 * npt
    u = rng_bits(seed, 2 * npt)
    th = 0.0 + (2.0 * 3.14159265358979323846 - 0.0) * u[0::2]
    ph = 0.0 + (3.14159265358979323846 - 0.0) * u[1::2]
    start = np.empty(n)
    start[0::3] = np.cos(th) * np.sin(ph)
    start[1::3] = np.sin(th) * np.sin(ph)
    start[2::3] = np.cos(ph)
    hp_ptr = np.zeros(n + 1, np.int32)
    hp_ptr[1:] = np.cumsum(np.arange(n, 0, -1))
    hp_idx = np.concatenate([np.arange(c, n, dtype=np.int32) for c in range(n)])
    jp_ptr = (3 * np.arange(npt + 1)).astype(np.int32)
    jp_idx = np.arange(n, dtype=np.int32)
    inst = Instance(f"elec:{npt}:{seed}", n, 0, npt, npt, hp_ptr, hp_idx, jp_ptr, jp_idx,
                    np.full(n, -np.inf), np.full(n, np.inf), start)
    inst.evaluator = _ElecEval(npt, inst)
    return inst


class _BearingEval:
    """COPS 3.0 'bearing' (journal bearing, b = 10, eps = 0.1): pressure v >= 0
    on an nx x ny interior grid of [0, 2 pi] x [0, 2b], v = 0 on the boundary,
    minimising sum_edges 0.5 hx hy wq (dv/dh)^2 - hx hy sum_nodes wl v with
    wq = (1 + eps cos xi)^3 (at edge midpoints), wl = eps sin xi.  Quadratic:
    the Hessian is the constant weighted 5-point stencil; no constraints (m = 0,
    so K2r = K1s = H + Sigma + delta I).  Not in the reference (SURVEY.md 8(d)
    config #2): a repo generator of the COPS shape."""

    def __init__(self, nx, ny, inst):
        b, eps = 10.0, 0.1
        self.nx, self.ny = nx, ny
        hx, hy = 2.0 * np.pi / (nx + 1), 2.0 * b / (ny + 1)
        xi = hx * np.arange(1, nx + 1)
        wq_mid = (1.0 + eps * np.cos(hx * (np.arange(nx + 1) + 0.5))) ** 3   # x-edges i -> i+1 (i = 0..nx)
        wq_node = (1.0 + eps * np.cos(xi)) ** 3                            # y-edges at column xi
        ax = hy / hx * wq_mid              # weight of an x-edge
        ay = hx / hy * wq_node             # weight of a y-edge (per column)
        n = nx * ny
        diag = np.zeros(n)
        I = np.arange(nx)
        for j in range(ny):
            c = j * nx + I
            diag[c] += ax[I] + ax[I + 1] + 2.0 * ay[I]
        self.diag = diag
        self.offx = -ax[1:nx]              # (i, i+1) inside a grid row
        self.offy = -ay                    # (j, j+1) per column i
        self.lin = -hx * hy * eps * np.sin(xi)
        self.inst = inst

    def hval(self):
        nx, ny = self.nx, self.ny
        ptr = self.inst.hp_ptr
        c = np.arange(nx * ny)
        i, j = c % nx, c // nx
        hx_, hy_ = i + 1 < nx, j + 1 < ny
        h = np.empty(int(ptr[-1]))
        h[ptr[:-1]] = self.diag
        h[ptr[:-1][hx_] + 1] = self.offx[i[hx_]]
        h[ptr[:-1][hy_] + 1 + hx_[hy_]] = self.offy[i[hy_]]
        return h

    def eval(self, t, y):
        import scipy.sparse as sp
        h = self.hval()
        n = len(t)
        ip, ix = self.inst.hp_ptr, self.inst.hp_idx
        L = sp.csc_matrix((h, ix, ip), shape=(n, n))
        g = L @ t + L.T @ t - h[ip[:-1]] * t   # symmetric product from the lower triangle
        return h, np.zeros(0), g + np.tile(self.lin, self.ny), np.zeros(0)


def bearing(nx: int, ny: int) -> Instance:
    n = nx * ny
    c = np.arange(n)
    has_x, has_y = (c % nx) + 1 < nx, (c // nx) + 1 < ny
    cnt = 1 + has_x.astype(np.int32) + has_y.astype(np.int32)
    hp_ptr = np.zeros(n + 1, np.int32)
    hp_ptr[1:] = np.cumsum(cnt)
    hp_idx = np.empty(int(hp_ptr[-1]), np.int32)
    hp_idx[hp_ptr[:-1]] = c
    hp_idx[hp_ptr[:-1][has_x] + 1] = c[has_x] + 1
    hp_idx[hp_ptr[:-1][has_y] + 1 + has_x[has_y]] = c[has_y] + nx
    inst = Instance(f"bearing:{nx}:{ny}", n, 0, 0, 0, hp_ptr, hp_idx, np.zeros(1, np.int32),
                    np.zeros(0, np.int32), np.zeros(n), np.full(n, np.inf), np.full(n, 0.5))
    inst.evaluator = _BearingEval(nx, ny, inst)
    return inst

def rng_bits(seed: int, k: int) -> np.ndarray:
    """k draws of problems.cpp:20-23's u = (gen() >> 11) * 2^-53"""
    g = MT19937_64(seed)
    return (g.raw(k) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def build(spec: str) -> Instance:
    t = spec.split(":")
    if t[0] == "opf_toy":
        return opf_toy(int(t[1]), int(t[2]))
    if t[0] == "opf_mesh":
        return opf_mesh(int(t[1]), int(t[2]), int(t[3]))
    if t[0] == "mpcc_sep":
        return mpcc_sep(int(t[1]))
    if t[0] == "elec":
        return elec(int(t[1]), int(t[2]))
    if t[0] == "bearing":
        return bearing(int(t[1]), int(t[2]))
    raise ValueError(f"unknown instance spec {spec}")


def kkt_case(inst: Instance, seed: int, rho: float = 100.0):
    """proj/tests/test_kkt.cpp:40-68: t = start + U(-.05,.05), y ~ U(-.01,.01)
    -> hval, jval; sigma ~ U(.5,2), rbar1 ~ U(-1,1) (n), rbar2, rbar3 ~ U(-1,1)
    (m).  Returns a dict of the KktInput arrays."""
    rng = MT19937_64(seed)
    t = inst.start + rng.uniform(-0.05, 0.05, inst.nt)
    y = rng.uniform(-0.01, 0.01, inst.m)
    hval, jval, _, _ = inst.evaluator.eval(t, y)
    n, m = inst.n, inst.m
    return dict(hval=hval, jval=jval, sigma=rng.uniform(0.5, 2.0, n),
                rbar1=rng.uniform(-1.0, 1.0, n), rbar2=rng.uniform(-1.0, 1.0, m),
                rbar3=rng.uniform(-1.0, 1.0, m), rho=rho)
