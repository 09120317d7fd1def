"""Raw-metric + stall-reason summary of one ncu report (python tools/ncu_summary.py rep out.txt)."""
import csv, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw)); hdr = rows[0]; d = dict(zip(hdr, rows[2]))
keys = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum', 'launch__grid_size', 'launch__block_size',
        'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'lts__t_sector_hit_rate.pct']
lines = [f"{k} {d.get(k)}" for k in keys if k in d]
items = []
for k in hdr:
    if 'smsp__pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued'):
        try: items.append((float(d[k].replace(',', '')), k))
        except ValueError: pass
items.sort(reverse=True); tot = sum(v for v, _ in items) or 1
lines.append("stall reasons (pc sampling):")
lines += [f"  {100 * v / tot:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}" for v, k in items[:8]]
open(out, "w").write("\n".join(lines) + "\n"); print("\n".join(lines))
