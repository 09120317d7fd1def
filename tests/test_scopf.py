"""SCOPF sharding: contingency blocks over ranks, Schur
complement of the coupling set-points summed with collectives.

CPU (no GPU): the generator's shares partition the global problem; the ranks'
K1s matrices (the oracle's bit-exact refill, kkt.cpp:149-186) sum to the
global one; and a world-size-2 gloo run of the distributed protocol (owner
conventions, delta correction, Schur / rhs / inertia sums) restated in numpy
reproduces the global oracle's step and delta decisions.
GPU: the sm_100a Schur-mode path (ncl_schur_*) in one process and in two
processes (gloo on one device), against the oracle's KktContext::solve on the
whole matrix: identical delta / attempts / perturbed decisions, step within
1e-8 relative (STEP_RTOL of test_gpu_kkt.py).
"""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_05885_b200 import scopf as SC

STEP_RTOL = 1e-8
KEYS = ("hval", "jval", "sigma", "rbar1", "rbar2", "rbar3")


def problem(inst):
    return O.Problem(inst.name, inst.nt, inst.ns, inst.m_eq, inst.m, inst.hp_ptr, inst.hp_idx,
                     inst.jp_ptr, inst.jp_idx)


def kcase(c):
    return O.KktCase(*(c[k] for k in KEYS), c["rho"])


def indefinite(c, s=-3.0):
    """scale the Hessian so the delta loop escalates (kkt.cpp:273-313)"""
    c = dict(c)
    c["hval"] = c["hval"] * s
    return c


def global_ref(D, seed, transform=None, warm=0.0):
    G = SC.subproblem(D, 0, D.K, True)
    c = SC.scopf_case(G, seed)
    if transform:
        c = transform(c)
    return G, c, O.OrcKkt(problem(G), "k1s").solve(kcase(c), warm)


def test_shares_partition_the_global_problem():
    D = SC.scopf_data(24, 7, 11)
    G = SC.subproblem(D, 0, D.K, True)
    c = SC.scopf_case(G, 3)
    assert G.m_eq == D.K * D.nbus and G.nt == D.nbus * (1 + 2 * D.K)
    for W in (1, 2, 3, 7):
        acc = {k: np.zeros_like(c[k]) for k in KEYS}
        nt_sum = 0
        for g in range(W):
            k0, k1 = SC.block_range(D.K, W, g)
            sub = SC.subproblem(D, k0, k1, g == 0)
            cs = SC.scopf_case(sub, 3)
            tmap, smap, rmap = SC.global_maps(D, sub, G)
            nmap = np.concatenate([tmap, G.nt + smap])
            for k in ("sigma", "rbar1"):
                np.add.at(acc[k], nmap, cs[k])
            for k in ("rbar2", "rbar3"):
                acc[k][rmap] += cs[k]
            nt_sum += sub.nt - sub.scopf["n0"]
            # the share's Jacobian / Hessian entries are the global ones
            for r in range(sub.m):
                gr = rmap[r]
                cols = tmap[sub.jp_idx[sub.jp_ptr[r]:sub.jp_ptr[r + 1]]]
                assert np.array_equal(cols, G.jp_idx[G.jp_ptr[gr]:G.jp_ptr[gr + 1]])
                assert np.array_equal(cs["jval"][sub.jp_ptr[r]:sub.jp_ptr[r + 1]],
                                      c["jval"][G.jp_ptr[gr]:G.jp_ptr[gr + 1]])
        assert nt_sum + D.nbus == G.nt
        for k in ("sigma", "rbar1", "rbar2", "rbar3"):
            assert np.array_equal(acc[k], c[k]), k


def test_k1s_is_block_arrowhead():
    D = SC.scopf_data(20, 5, 2)
    G = SC.subproblem(D, 0, D.K, True)
    cp, ri, _ = O.OrcKkt(problem(G), "k1s").matrix()
    nb = D.nbus
    blk = lambda v: -1 if v < nb else (v - nb) // (2 * nb)
    for j in range(G.nt):
        for p in range(cp[j], cp[j + 1]):
            a, b = blk(ri[p]), blk(j)
            assert a == b or a == -1 or b == -1


def embed_sum(D, W, seed, delta, transform=None):
    """sum over ranks of the shares' refilled K1s, in global indexing (dense)"""
    G = SC.subproblem(D, 0, D.K, True)
    tot = np.zeros((G.nt, G.nt))
    for g in range(W):
        k0, k1 = SC.block_range(D.K, W, g)
        sub = SC.subproblem(D, k0, k1, g == 0)
        cs = SC.scopf_case(sub, seed)
        if transform:
            cs = transform(cs)
        Q = O.OrcKkt(problem(sub), "k1s")
        cp, ri, v = Q.matrix()
        v = Q.refill(kcase(cs), delta)
        tmap, _, _ = SC.global_maps(D, sub, G)
        for j in range(sub.nt):
            for p in range(cp[j], cp[j + 1]):
                i = ri[p]
                tot[tmap[i], tmap[j]] += v[p]
                if i != j:
                    tot[tmap[j], tmap[i]] += v[p]
    return G, tot


@pytest.mark.parametrize("W", [2, 3])
def test_rank_matrices_sum_to_the_global_k1s(W):
    D = SC.scopf_data(18, 5, 9)
    delta = 3e-4
    G, tot = embed_sum(D, W, 4, delta)
    n0 = D.nbus
    tot[np.arange(n0), np.arange(n0)] -= (W - 1) * delta  # delta counts once
    Q = O.OrcKkt(problem(G), "k1s")
    cp, ri, _ = Q.matrix()
    v = Q.refill(kcase(SC.scopf_case(G, 4)), delta)
    ref = np.zeros_like(tot)
    for j in range(G.nt):
        for p in range(cp[j], cp[j + 1]):
            ref[ri[p], j] = ref[j, ri[p]] = v[p]
    assert np.abs(tot - ref).max() <= 1e-13 * np.abs(ref).max()


# --------------------------------------------------------------------------
# the collective protocol of ScopfKkt, restated in numpy (dense per rank)
def _inertia(M):
    ev = np.linalg.eigvalsh(M)
    return int((ev > 0).sum()), int((ev < 0).sum())


def _dist_worker(rank, world, port, nbus, K, seed, scale, out):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    D = SC.scopf_data(nbus, K, seed)
    G = SC.subproblem(D, 0, K, True)
    k0, k1 = SC.block_range(K, world, rank)
    sub = SC.subproblem(D, k0, k1, rank == 0)
    cs = SC.scopf_case(sub, 5)
    cs["hval"] = cs["hval"] * scale
    Q = O.OrcKkt(problem(sub), "k1s")
    cp, ri, _ = Q.matrix()
    n0, N = sub.scopf["n0"], sub.nt
    allsum = lambda a: (dist.all_reduce(t := torch.from_numpy(np.ascontiguousarray(a))), t.numpy())[1]
    allmax = lambda v: (dist.all_reduce(t := torch.tensor([v]), op=dist.ReduceOp.MAX), float(t[0]))[1]
    hmax = allmax(max(np.abs(cs["hval"]).max(), np.abs(cs["sigma"]).max()))
    delta, first, att = 0.0, True, 0
    while True:
        att += 1
        v = Q.refill(kcase(cs), delta)
        A = np.zeros((N, N))
        for j in range(N):
            for p in range(cp[j], cp[j + 1]):
                A[ri[p], j] = A[j, ri[p]] = v[p]
        Abb, Ab0, A00 = A[n0:, n0:], A[n0:, :n0], A[:n0, :n0]
        Sg = A00 - Ab0.T @ np.linalg.solve(Abb, Ab0)
        pos, neg = _inertia(Abb)
        S = allsum(Sg) - (world - 1) * delta * np.eye(n0)
        cnt = allsum(np.array([pos, neg], np.float64))
        ps, ns_ = _inertia(S)
        if cnt[0] + ps == G.nt and cnt[1] + ns_ == 0:
            b = Q.build_rhs(kcase(cs), delta)
            bb, b0 = b[n0:], b[:n0]
            rb = b0 - Ab0.T @ np.linalg.solve(Abb, bb)
            x0 = np.linalg.solve(S, allsum(rb))
            xb = np.linalg.solve(Abb, bb - Ab0 @ x0)
            out[rank] = (delta, att, np.concatenate([x0, xb]))
            break
        delta = (1e-8 * max(1.0, hmax)) if first else delta * 8.0
        first = False
    dist.destroy_process_group()


@pytest.mark.parametrize("scale", [1.0, -3.0])
def test_collective_protocol_world2_gloo(scale):
    """world_size 2 over gloo on CPU: the same sums / corrections / delta loop
    as ScopfKkt, dense numpy per rank; the t-part of the step equals the
    global oracle's (K1s solution = dt)."""
    import torch.multiprocessing as mp
    nbus, K, seed = 16, 5, 6
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_dist_worker, args=(2, port, nbus, K, seed, scale, out), nprocs=2, join=True)
    D = SC.scopf_data(nbus, K, seed)
    G, c, ref = global_ref(D, 5, transform=lambda c: indefinite(c, scale))
    assert ref.ok
    for rank in range(2):
        delta, att, x = out[rank]
        assert delta == ref.delta and att == ref.factor_attempts
        k0, k1 = SC.block_range(K, 2, rank)
        sub = SC.subproblem(D, k0, k1, rank == 0)
        tmap, _, _ = SC.global_maps(D, sub, G)
        sc = max(1.0, np.abs(ref.dx).max())
        assert np.abs(x - ref.dx[:G.nt][tmap]).max() <= 1e-9 * sc
    if scale < 0:
        assert ref.factor_attempts > 1


# --------------------------------------------------------------------------
def _gpu_check(st, ref, D, sub, G):
    assert (bool(st["ok"]), st["factor_attempts"], st["delta"], st["perturbed_pivots"]) == \
        (ref.ok, ref.factor_attempts, ref.delta, ref.perturbed_pivots)
    tmap, smap, rmap = SC.global_maps(D, sub, G)
    nmap = np.concatenate([tmap, G.nt + smap])
    sc = max(1.0, np.abs(ref.dx).max(), np.abs(ref.dy).max())
    for k, m in (("dx", nmap), ("dr", rmap), ("dy", rmap)):
        assert np.abs(st[k].cpu().numpy() - getattr(ref, k)[m]).max() <= STEP_RTOL * sc, k


@pytest.mark.gpu
@pytest.mark.parametrize("nbus,K,seed,scale", [(30, 8, 3, 1.0), (118, 12, 4, 1.0), (40, 6, 2, -3.0),
                                                 (14, 140, 5, 1.0)])  # >= 128 blocks: split extend-add
def test_gpu_schur_single_rank_matches_oracle(nbus, K, seed, scale):
    import torch
    D = SC.scopf_data(nbus, K, seed)
    G, c, ref = global_ref(D, 5, transform=lambda c: indefinite(c, scale))
    cs = c
    dev = {k: torch.tensor(cs[k], dtype=torch.float64, device="cuda") for k in KEYS}
    st = SC.ScopfKkt(G, G.nt).solve(dev, cs["rho"], 0.0)
    _gpu_check(st, ref, D, G, G)


def _gpu_worker(rank, world, port, nbus, K, seed, scale, out):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    D = SC.scopf_data(nbus, K, seed)
    k0, k1 = SC.block_range(K, world, rank)
    sub = SC.subproblem(D, k0, k1, rank == 0)
    cs = indefinite(SC.scopf_case(sub, 5), scale)
    dev = {k: torch.tensor(cs[k], dtype=torch.float64, device="cuda") for k in KEYS}
    G = SC.subproblem(D, 0, K, True)
    st = SC.ScopfKkt(sub, G.nt, dist=dist).solve(dev, cs["rho"], 0.0)
    out[rank] = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in st.items()}
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [1.0, -3.0])
def test_gpu_schur_two_ranks_gloo_matches_oracle(scale):
    """two processes sharing the device, gloo collectives (NCCL needs one GPU
    per rank; the collective calls are the same)"""
    import torch
    import torch.multiprocessing as mp
    nbus, K, seed = 30, 9, 3
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gpu_worker, args=(2, port, nbus, K, seed, scale, out), nprocs=2, join=True)
    D = SC.scopf_data(nbus, K, seed)
    G, c, ref = global_ref(D, 5, transform=lambda c: indefinite(c, scale))
    for rank in range(2):
        k0, k1 = SC.block_range(K, 2, rank)
        sub = SC.subproblem(D, k0, k1, rank == 0)
        st = {k: (torch.from_numpy(v) if isinstance(v, np.ndarray) else v) for k, v in out[rank].items()}
        _gpu_check(st, ref, D, sub, G)
