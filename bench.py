#!/usr/bin/env python
"""Benchmark of the Newton-step hot path (one ``KktContext::solve``: refill,
static-pivot LDL^T with inertia/delta control, refined solve, recovery) on
B200.

One JSON line (rank 0).  ``value`` = milliseconds per Newton step with the
inputs resident in HBM (device-pointer C-ABI call); ``e2e`` = the same through
the host-buffer C-ABI call (``ncl_kkt_solve``: H2D of hval/jval/sigma/rbar,
D2H of dx/dr/dy inside the timed region).  ``roofline`` is the dominant phase
of the step measured live with CUDA events on the context's stream;
``cpu_baseline`` times the reference's own KktContext (compiled unmodified
from proj/src, oracle/_ref/libncl_ref.so) or the C restatement on one host
core.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload opf_mesh:280:280:1] [--form k1s]

Multi-GPU: a single ACOPF instance does not shard: N ranks
run N independent replicas ("replicas only", weak scaling); the job time is
the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_WORKLOAD = "opf_mesh:280:280:1"  # 78,400 buses: BASELINE config #3, mesh variant
METRIC = "KKT factor+solve ms/iter (NCL Newton step, KktContext::solve)"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- workload
def make_workload(spec, seed=42, world=1):
    if spec.startswith("scopf:"):  # the whole problem of `world` ranks' blocks
        from paper_2510_05885_b200 import scopf as SC
        nbus, kp, sd = SC.parse_spec(spec)
        D = SC.scopf_data(nbus, kp * world, sd)
        inst = SC.subproblem(D, 0, D.K, True)
        return inst, SC.scopf_case(inst, seed)
    from paper_2510_05885_b200 import instances as I
    inst = I.build(spec)
    case = I.kkt_case(inst, seed)
    return inst, case


def algorithmic_work(info, inst, form):
    """SURVEY.md 8(d) per-unit formulas (bytes, flops)."""
    N, nnzA, lnz = info.n, info.nnz, info.l_nnz
    n, m = inst.n, inst.m
    hnnz, jnnz = len(inst.hp_idx), len(inst.jp_idx)
    return dict(
        assemble=(8.0 * (hnnz + jnnz + n + m + nnzA),
                  3.0 * info.npairs + hnnz + inst.nt if form == "k1s" else float(n + m)),
        factor=(8.0 * (nnzA + lnz + N), float(info.flops)),
        solve=(24.0 * lnz + 40.0 * N, 4.0 * lnz + N),
        matvec=(12.0 * nnzA + 24.0 * N, 4.0 * nnzA),
    )


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every ~2 ms through
    NVML while the timed region runs (the recipe's clocks line); nvidia-smi
    -lms polling as the fallback."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.reasons = [], None, set()
        self.stop_evt = threading.Event()
        self.t = None

    def _run(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        while True:
            self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
            r = int(get_r(h))
            for k, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(k)
            if self.stop_evt.wait(0.002):
                break
        pynvml.nvmlShutdown()

    def start(self):
        try:
            import pynvml  # noqa: F401
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None

    def stop(self):
        self.stop_evt.set()
        if self.t:
            self.t.join(timeout=2)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ------------------------------------------------------------- CPU baselines
def cpu_reference_run(inst, case, form, n_solves, budget_s):
    """The reference's own KktContext (proj/src/kkt.cpp, compiled unmodified)
    if its library is present, else the C restatement; one host core."""
    from oracle import oracle as O
    from tests_helpers_shim import problem_case
    prob, kcase = problem_case(inst, case)
    kind = "reference" if O.ref_available() else "port"
    ctx = O.RefKkt(prob, form) if kind == "reference" else O.OrcKkt(prob, form)
    times = []
    t_start = time.perf_counter()
    for _ in range(max(1, n_solves)):
        t0 = time.perf_counter()
        st = ctx.solve(kcase, 0.0)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    return kind, times, st


def measure_fp64_peak(torch):
    """DGEMM (cuBLAS, FP64 tensor cores) burst throughput, TFLOP/s."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


# ------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--form", default="k1s", choices=["k1s", "k2r", "k2"])
    ap.add_argument("--cpu-budget", type=float, default=25.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return reference_arm(args, world, rank)
    if args.workload.startswith("scopf:"):
        return scopf_bench(args, world, rank, local)

    import torch
    import torch.distributed as dist
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)

    import paper_2510_05885_b200 as P
    inst, case = make_workload(args.workload)
    hp = P.HessianPattern(inst.nt, inst.hp_ptr, inst.hp_idx)
    jp = P.JacobianPattern(inst.m, inst.nt, inst.jp_ptr, inst.jp_idx)
    t0 = time.perf_counter()
    ctx = P.KktContext(hp, jp, inst.nt, inst.ns, inst.m_eq, P.parse_kkt_form(args.form))
    t_symbolic = time.perf_counter() - t0
    info = ctx.info
    keys = ("hval", "jval", "sigma", "rbar1", "rbar2", "rbar3")
    dev = {k: torch.tensor(case[k], dtype=torch.float64, device="cuda") for k in keys}
    outs = [torch.zeros(max(1, n), dtype=torch.float64, device="cuda") for n in (inst.n, inst.m, inst.m)]
    ptrs = [dev[k].data_ptr() for k in keys]
    optrs = [t.data_ptr() for t in outs]
    stream = torch.cuda.ExternalStream(ctx.stream())
    flush = torch.empty(384 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def solve_dev():
        st = ctx.solve_device(ptrs, case["rho"], 0.0, optrs)
        if not st.ok:
            raise RuntimeError("KKT solve failed on the benchmark workload")
        return st

    for _ in range(max(3, args.warmup)):
        st = solve_dev()
    torch.cuda.synchronize()

    # ------------------------------------------------ timed region (device)
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    ctx.set_timing(True)
    l0 = ctx.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = 0.0
    phase = np.zeros(4)
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (outside the events)
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        st = solve_dev()
        e.record(stream)
        e.synchronize()
        total_ms += s.elapsed_time(e)
        t = ctx.last_timing()
        phase += [t["assemble_ms"], t["factor_ms"], t["solve_ms"], t["recover_ms"]]
    torch.cuda.synchronize()
    launches = ctx.launch_count() - l0
    ctx.set_timing(False)
    if world > 1:
        dist.barrier()
        tt = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    clk = clocks.stop()
    ms_per_step = total_ms / args.steps
    # ms per Newton step (max over ranks): every rank solves its own replica,
    # so the job's latency per step is the slowest rank's; the replicas'
    # combined rate is reported beside it (job_steps_per_s)
    value = ms_per_step

    # ------------------------------------------------ e2e (host buffers)
    pinned = {k: torch.tensor(case[k], dtype=torch.float64).pin_memory() for k in keys}
    host_in = P.KktInput(*[pinned[k].numpy() for k in keys], case["rho"])
    host_out = tuple(torch.zeros(n, dtype=torch.float64).pin_memory().numpy() for n in (inst.n, inst.m, inst.m))
    e2e_ms = 0.0
    ctx.solve(host_in, 0.0, out=host_out)
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        stp = ctx.solve(host_in, 0.0, out=host_out)
        e.record(stream)
        e.synchronize()
        e2e_ms += s.elapsed_time(e)
        assert stp.ok
    if world > 1:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    h2d = 8 * sum(len(case[k]) for k in keys)
    d2h = 8 * (inst.n + 2 * inst.m)

    # ------------------------------------------------ roofline (live)
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback"
    fp64_peak = measure_fp64_peak(torch) if rank == 0 else 0.0
    work = algorithmic_work(info, inst, args.form)
    per = phase / args.steps
    names = ["assemble", "factor", "solve", "recover"]
    dom = int(np.argmax(per))
    refine = st.refine_steps
    if names[dom] == "factor":
        b, fl = work["factor"]
        b *= st.factor_attempts
        fl *= st.factor_attempts
    elif names[dom] == "solve":
        b = (1 + refine) * work["solve"][0] + (1 + refine) * work["matvec"][0]
        fl = (1 + refine) * work["solve"][1] + (1 + refine) * work["matvec"][1]
    elif names[dom] == "assemble":
        b, fl = work["assemble"]
    else:
        b, fl = 8.0 * (inst.n + 2 * inst.m + len(inst.jp_idx)), 0.0
    t_dom = per[dom] / 1e3
    ach_gbs = b / t_dom / 1e9
    ach_tf = fl / t_dom / 1e12
    frac_hbm = ach_gbs / hbm_peak
    frac_fp = ach_tf / fp64_peak if fp64_peak > 0 else 0.0
    use_tensor = fp64_peak > 0 and (fl / (fp64_peak * 1e12)) > (b / (hbm_peak * 1e9))
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get(f"{args.workload}/{args.form}/{names[dom]}")
        except Exception:
            traffic = None
    roofline = {
        "bound": "tensor" if use_tensor else "hbm",
        "kernel": f"{names[dom]} phase ({'warp-tier + wide-tier LDL^T kernels' if names[dom] == 'factor' else names[dom]})",
        "achieved": round(ach_tf if use_tensor else ach_gbs, 4),
        "peak": round(fp64_peak if use_tensor else hbm_peak, 2),
        "unit": "TFLOP/s" if use_tensor else "GB/s",
        "frac": round(frac_fp if use_tensor else frac_hbm, 5),
        "traffic": traffic,
        "peak_source": ("FP64 DGEMM measured live in this run (cuBLAS, float64)" if use_tensor
                        else f"HBM copy {hbm_src}"),
        "algorithmic_bytes": b, "algorithmic_flops": fl,
        "hbm_frac": round(frac_hbm, 5), "fp64_frac": round(frac_fp, 5),
        "fp64_peak_tflops": round(fp64_peak, 2),
        "phase_ms": {k: round(v, 4) for k, v in zip(names, per)},
    }

    # ------------------------------------------------ CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        kind, times, cst = cpu_reference_run(inst, case, args.form, 50, args.cpu_budget)
        cpu = {"value": round(1e3 * float(np.mean(times)), 3), "unit": "ms/iter", "cores": 1,
               "kind": kind,
               "sample": f"{len(times)} KktContext::solve calls on {args.workload} ({args.form}), "
                         f"single thread, {'reference kkt.cpp+sparse.cpp compiled unmodified' if kind == 'reference' else 'C restatement'}",
               "host_cpu": host_cpu()}

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 4), "unit": "ms/iter", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded reference-recipe KKT inputs, test_kkt.cpp:40-68)",
            "config": {"workload": args.workload, "kkt_form": args.form, "N": info.n, "nnz_K": info.nnz,
                       "nnz_L": info.l_nnz, "factor_flops": info.flops, "supernodes": info.n_supernodes,
                       "sn_height": info.sn_height, "wide_fronts": info.n_wide, "wide_levels": info.n_levels,
                       "max_front": info.max_front, "parallelism": f"replicas x{world}",
                       "l2": "flushed between timed steps (384 MiB write)",
                       "factor_attempts": st.factor_attempts, "refine_steps": st.refine_steps,
                       "symbolic_once_s": round(t_symbolic, 3)},
            "job_steps_per_s": round(1e3 * world / ms_per_step, 2),
            "e2e": {"value": round(e2e_ms / args.steps, 4), "unit": "ms/iter",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def scopf_bench(args, world, rank, local):
    """SCOPF (BASELINE config #5): scopf:<nbus>:<blocks per GPU>:<seed>, weak
    scaling -- rank g owns blocks [g*Kp, (g+1)*Kp) of one global problem and
    every step is ONE distributed KktContext::solve of the whole system
    (Schur complement of the coupling set-points all-reduced over NCCL)."""
    import torch
    import torch.distributed as dist
    from paper_2510_05885_b200 import scopf as SC
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    nbus, kp, sd = SC.parse_spec(args.workload)
    D = SC.scopf_data(nbus, kp * world, sd)
    k0, k1 = SC.block_range(D.K, world, rank)
    sub = SC.subproblem(D, k0, k1, rank == 0)
    case = SC.scopf_case(sub, 42)
    nt_global = nbus * (1 + 2 * D.K)
    keys = ("hval", "jval", "sigma", "rbar1", "rbar2", "rbar3")
    t0 = time.perf_counter()
    K = SC.ScopfKkt(sub, nt_global, dist=dist if world > 1 else None)
    t_symbolic = time.perf_counter() - t0
    dev = {k: torch.tensor(case[k], dtype=torch.float64, device="cuda") for k in keys}
    flush = torch.empty(384 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(max(3, args.warmup)):
        st = K.solve(dev, case["rho"], 0.0)
        assert st["ok"]
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        st = K.solve(dev, case["rho"], 0.0)
        e.record()
        e.synchronize()
        total_ms += s.elapsed_time(e)
    if world > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    clk = clocks.stop()
    # e2e: host (pinned) inputs copied in, the step copied out, every step
    pinned = {k: torch.tensor(case[k], dtype=torch.float64).pin_memory() for k in keys}
    host_out = None
    e2e_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dv = {k: pinned[k].to("cuda", non_blocking=True) for k in keys}
        stp = K.solve(dv, case["rho"], 0.0)
        if host_out is None:  # pinned result buffers (allocated once, outside the steady state)
            host_out = [torch.empty(stp[k].shape, dtype=torch.float64).pin_memory() for k in ("dx", "dr", "dy")]
        out = [h.copy_(stp[k], non_blocking=True) for h, k in zip(host_out, ("dx", "dr", "dy"))]
        e.record()
        e.synchronize()
        e2e_ms += s.elapsed_time(e)
        assert stp["ok"] and len(out) == 3
    if world > 1:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    import ctypes as C
    from paper_2510_05885_b200 import _lib
    info = _lib.KktInfo()
    _lib.lib().ncl_schur_info(K.h, C.byref(info))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        inst_g, case_g = make_workload(args.workload, world=1)
        kind, times, _ = cpu_reference_run(inst_g, case_g, "k1s", 50, args.cpu_budget)
        cpu = {"value": round(1e3 * float(np.mean(times)), 3), "unit": "ms/iter", "cores": 1, "kind": kind,
               "sample": f"{len(times)} KktContext::solve calls on the whole {args.workload} K1s system, "
                         "single thread", "host_cpu": host_cpu()}
    if rank == 0:
        value = total_ms / args.steps
        res = {
            "metric": METRIC, "value": round(value, 4), "unit": "ms/iter", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(value, 4),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic SCOPF (seeded, repo generator; per-block reference-recipe KKT inputs)",
            "config": {"workload": args.workload, "kkt_form": "k1s", "blocks_total": D.K,
                       "blocks_per_gpu": kp, "N_global": nt_global, "N_local": info.n,
                       "coupling_n0": nbus, "nnz_K_local": info.nnz, "factor_flops_local": info.flops,
                       "parallelism": f"contingency blocks sharded x{world}, Schur all-reduce",
                       "l2": "flushed between timed steps (384 MiB write)",
                       "factor_attempts": st["factor_attempts"], "refine_steps": st["refine_steps"],
                       "symbolic_once_s": round(t_symbolic, 3)},
            "e2e": {"value": round(e2e_ms / args.steps, 4), "unit": "ms/iter",
                    "h2d_bytes_per_step": 8 * sum(len(case[k]) for k in keys),
                    "d2h_bytes_per_step": 8 * (sub.n + 2 * sub.m)},
            "roofline": None,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


def host_cpu():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference_arm(args, world, rank):
    """--impl reference: the reference's own CPU KktContext on this box's host
    cores, same workload/metric/unit; rank 0 only."""
    if rank != 0:
        return
    inst, case = make_workload(args.workload, world=world)
    budget = max(30.0, min(150.0, 6.0 * args.steps))
    n_warm = max(1, args.warmup)  # the requested warm-up, bounded by the same time budget
    _, wt, _ = cpu_reference_run(inst, case, args.form, n_warm, budget)
    n_warm = len(wt)
    kind, times, st = cpu_reference_run(inst, case, args.form, args.steps, budget)
    v = 1e3 * float(np.mean(times))
    out = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms/iter", "n_gpus": world,
        "steps": len(times), "warmup": n_warm, "ms_per_step": round(v, 3), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded reference-recipe KKT inputs, test_kkt.cpp:40-68)",
        "config": {"workload": args.workload, "kkt_form": args.form, "parallelism": "1 host thread"},
        "cpu_baseline": {"value": round(v, 3), "unit": "ms/iter", "cores": 1, "kind": kind,
                         "sample": f"{len(times)} of {args.steps} requested steps (time budget {budget:.0f}s)",
                         "host_cpu": host_cpu()},
        "e2e": {"value": round(v, 3), "unit": "ms/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
