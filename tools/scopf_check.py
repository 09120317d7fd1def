"""Distributed SCOPF KKT solve vs the oracle's single-matrix KktContext
(diagnostic; the parity tests live in tests/test_scopf.py).

    python tools/scopf_check.py [nbus K seed]
    torchrun --nproc-per-node 2 tools/scopf_check.py 30 8 3 --backend gloo
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2510_05885_b200 import scopf as SC  # noqa: E402


def main():
    backend = "gloo" if "gloo" in sys.argv else "nccl"
    args = [a for a in sys.argv[1:] if not a.startswith("--") and a not in ("gloo", "nccl")]
    nbus, K, seed = (int(a) for a in args) if args else (30, 8, 3)
    dist = None
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) > 1:
        import torch.distributed as dist
        dist.init_process_group(backend)
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    world = dist.get_world_size() if dist else 1
    rank = dist.get_rank() if dist else 0
    D = SC.scopf_data(nbus, K, seed)
    G = SC.subproblem(D, 0, K, True)
    k0, k1 = SC.block_range(K, world, rank)
    sub = SC.subproblem(D, k0, k1, rank == 0)
    cs = SC.scopf_case(sub, 5)
    dev = {k: torch.tensor(cs[k], dtype=torch.float64, device="cuda") for k in
           ("hval", "jval", "sigma", "rbar1", "rbar2", "rbar3")}
    S = SC.ScopfKkt(sub, G.nt, dist=dist)
    st = S.solve(dev, cs["rho"], 0.0)
    case = SC.scopf_case(G, 5)
    prob = O.Problem(G.name, G.nt, G.ns, G.m_eq, G.m, G.hp_ptr, G.hp_idx, G.jp_ptr, G.jp_idx)
    ref = O.OrcKkt(prob, "k1s").solve(O.KktCase(case["hval"], case["jval"], case["sigma"], case["rbar1"],
                                                 case["rbar2"], case["rbar3"], case["rho"]), 0.0)
    tmap, smap, rmap = SC.global_maps(D, sub, G)
    nmap = np.concatenate([tmap, G.nt + smap])
    dx, dr, dy = (st[k].cpu().numpy() for k in ("dx", "dr", "dy"))
    sc = max(1.0, np.abs(ref.dx).max(), np.abs(ref.dy).max())
    err = max(np.abs(dx - ref.dx[nmap]).max(), np.abs(dr - ref.dr[rmap]).max(),
              np.abs(dy - ref.dy[rmap]).max()) / sc
    print(f"rank {rank}/{world}: ours delta {st['delta']} att {st['factor_attempts']} ref {st['refine_steps']} "
          f"pert {st['perturbed_pivots']} ok {st['ok']} | oracle delta {ref.delta} att {ref.factor_attempts} "
          f"ref {ref.refine_steps} pert {ref.perturbed_pivots} | step rel err {err:.3e}", flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
