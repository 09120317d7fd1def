"""Bitwise comparison of two library builds (tools/ab_lib.sh): solves one KKT
case with the library NCL_B200_LIB points at (or the in-tree one) and writes
dx | dr | dy to <out>.npy; `--compare a.npy b.npy` reports differing entries.

    NCL_B200_LIB=tools/ab/lib_head.so python tools/ab_bits.py opf_mesh:280:280:1 k1s gpurun_out/ab/head
    python tools/ab_bits.py opf_mesh:280:280:1 k1s gpurun_out/ab/tree
    python tools/ab_bits.py --compare gpurun_out/ab/head.npy gpurun_out/ab/tree.npy
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    d = int(np.count_nonzero(a.view(np.int64) != b.view(np.int64)))
    print(f"{d} of {a.size} entries differ bitwise" + ("" if d else " (identical)"))
    sys.exit(1 if d else 0)

from helpers import case_from_dict, gpu_context, gpu_input, problem_from_instance  # noqa: E402
from paper_2510_05885_b200 import instances as I  # noqa: E402

spec, form, out = sys.argv[1], sys.argv[2], sys.argv[3]
inst = I.build(spec)
case = case_from_dict(I.kkt_case(inst, 42))
ctx = gpu_context(problem_from_instance(inst), form)
r = ctx.solve(gpu_input(case), 0.0)
r = ctx.solve(gpu_input(case), 0.0)  # graphs replayed
np.save(out + ".npy", np.concatenate([r.dx, r.dr, r.dy]))
print(out, "ok" if r.ok else "FAILED")
