"""Aggregate ncu warp-stall samples per CUDA source line (needs -lineinfo).

    python tools_ncu_lines.py gpurun_out/prof.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname = "?"
    recs = []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if len(r) > 6 and r[0].isdigit() and r[2] == "-":
            try:
                recs.append((int(float(r[4])), fname, r[0], r[1].strip()[:90]))
            except ValueError:
                pass
    tot = sum(x[0] for x in recs)
    print("total samples", tot)
    for v, fn, ln, s in sorted(recs, key=lambda x: -x[0])[:top]:
        print(f"{v:6d} {100.0 * v / max(tot, 1):5.1f}%  {fn}:{ln}: {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
