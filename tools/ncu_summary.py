"""Summarise an ncu --set full capture (.ncu-rep) into the two text files kept
under profiles/: the key raw metrics of the launch, and the CUDA source lines
with the most warp-stall samples (the capture must be taken with
--import-source on and the kernels built with -lineinfo).

    python tools/ncu_summary.py <capture.ncu-rep> <out_prefix>
      -> <out_prefix>_raw_summary.txt, <out_prefix>_stall_lines.txt
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "sm__cycles_elapsed.avg",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_op_dmma.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "membar", "selected", "math_pipe_throttle",
          "mio_throttle", "lg_throttle", "no_instructions", "sleeping", "branch_resolving", "dispatch_stall",
          "drain", "imc_miss", "not_selected", "tex_throttle", "misc"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw_summary(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, vals = rows[0], rows[1], rows[2]
    out = []
    for m in METRICS:
        if m in h:
            i = h.index(m)
            out.append(f"{m:72s} {vals[i]} {units[i]}".rstrip())
    samp = {}
    for s in STALLS:
        m = f"smsp__pcsamp_warps_issue_stalled_{s}"
        if m in h:
            try:
                samp[s] = float(vals[h.index(m)].replace(",", ""))
            except ValueError:
                pass
    tot = sum(samp.values())
    if tot:
        out.append("")
        out.append("warp-stall samples (share of all sampled stall reasons):")
        for s, v in sorted(samp.items(), key=lambda x: -x[1]):
            if v:
                out.append(f"  {s:24s} {v:10.0f}  {100 * v / tot:5.1f}%")
    return "\n".join(out) + "\n"


def stall_lines(rep, top=30):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    cur, agg, src = None, collections.Counter(), {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        try:
            ln = int(r[0])
            v = float(r[4]) if len(r) > 4 and r[4] else 0.0
        except ValueError:
            continue
        agg[(cur, ln)] += v
        if r[1].strip():
            src[(cur, ln)] = r[1].strip()
    tot = sum(agg.values()) or 1.0
    out = [f"{'file:line':28s} {'stall %':>7s}  source"]
    for (f, ln), v in agg.most_common(top):
        out.append(f"{f + ':' + str(ln):28s} {100 * v / tot:6.1f}%  {src.get((f, ln), '')[:110]}")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    rep, prefix = sys.argv[1], sys.argv[2]
    open(prefix + "_raw_summary.txt", "w").write(raw_summary(rep))
    open(prefix + "_stall_lines.txt", "w").write(stall_lines(rep))
