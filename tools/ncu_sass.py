"""Per-SASS-instruction warp-stall samples from an ncu report (measurement aid).

    python tools/ncu_sass.py report.ncu-rep [min_samples]
Prints instructions with >= min_samples samples and their dominant stall reasons.
"""
import csv
import io
import subprocess
import sys


def main(rep, thr=1):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    tot = 0
    recs = []
    for r in rows:
        if len(r) > 5 and r[0] == "Address":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        try:
            n = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        tot += n
        st = sorted(((int(d[k]), k[6:]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k
                     and d[k].isdigit()), reverse=True)[:3]
        recs.append((d["Address"][-5:], d["Source"].strip()[:60], n, st))
    print("total samples", tot)
    for a, s, n, st in recs:
        if n >= thr:
            print(f"{a} {n:5d} {s:60s} " + " ".join(f"{k}:{v}" for v, k in st if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
