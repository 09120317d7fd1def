"""Summarise an ncu launch list per kernel: launches, device time and DRAM
traffic per solve (metrics gpu__time_duration.sum [+ dram__bytes_read.sum,
dram__bytes_write.sum]).

    python tools/launches.py gpurun_out/launches.csv <solves in the capture> [--json out.json]
"""
import collections
import re
import csv
import json
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi, gi, mi, idi = (h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size'),
                           h.index('Metric Name'), h.index('ID'))
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        try:
            v = float(r[vi].replace(',', ''))
        except (ValueError, IndexError):
            continue
        nm = re.sub(r'^(void )?(nclb::)?(<unnamed>::|\(anonymous namespace\)::)?', '', r[ki]).split('(')[0].strip()
        d = launches.setdefault(r[idi], {"name": nm, "grid": r[gi]})
        d[r[mi]] = v
    return list(launches.values())


def main(path, nsolves, out_json=None):
    L = load(path)
    t = collections.defaultdict(float)
    b = collections.defaultdict(float)
    c = collections.Counter()
    for d in L:
        n = d["name"]
        t[n] += d.get("gpu__time_duration.sum", 0.0)
        b[n] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        c[n] += 1
    ours = sum(v for k, v in t.items() if k.startswith('k_'))
    print(f"{'kernel':24s} {'launches':>9s} {'ms/solve':>9s} {'share':>7s} {'DRAM MB/solve':>14s} {'GB/s':>8s}")
    summary = {}
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        if not k.startswith('k_'):
            continue
        ms = v / 1e6 / nsolves
        mb = b[k] / 1e6 / nsolves
        gbs = (b[k] / v) if v else 0.0
        print(f"{k:24s} {c[k] / nsolves:9.1f} {ms:9.3f} {100 * v / ours:6.1f}% {mb:14.2f} {gbs:8.1f}")
        summary[k] = dict(launches_per_solve=c[k] / nsolves, ms_per_solve=ms, share=v / ours,
                          dram_bytes_per_solve=b[k] / nsolves)
    print(f"{'TOTAL (ours)':24s} {sum(v for k, v in c.items() if k.startswith('k_')) / nsolves:9.1f} "
          f"{ours / 1e6 / nsolves:9.3f}")
    if out_json:
        json.dump(summary, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    oj = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    if oj in args:
        args.remove(oj)
    main(args[0], float(args[1]) if len(args) > 1 else 1.0, oj)
