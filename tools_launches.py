"""Summarise an ncu launch list (gpu__time_duration per launch) per kernel."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
    out = []
    for r in rows[hi + 1:]:
        try:
            out.append((r[ki].split('(')[0].replace('nclb::', ''), float(r[vi].replace(',', '')), r[gi]))
        except (ValueError, IndexError):
            pass
    return out


def main(path, nsolves):
    L = load(path)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, v, _ in L:
        tot[n] += v
        cnt[n] += 1
    ours = sum(v for k, v in tot.items() if k.startswith('k_'))
    print(f"{'kernel':32s} {'launches':>9s} {'ms/solve':>9s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        if not k.startswith('k_'):
            continue
        print(f"{k:32s} {cnt[k] / nsolves:9.1f} {v / 1e6 / nsolves:9.3f} {100 * v / ours:6.1f}%")
    print(f"{'TOTAL (ours)':32s} {sum(c for k, c in cnt.items() if k.startswith('k_')) / nsolves:9.1f} {ours / 1e6 / nsolves:9.3f}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
