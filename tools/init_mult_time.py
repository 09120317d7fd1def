"""Time init_multipliers (solver.cpp:43-91): device path (ncl_init_multipliers)
vs the reference algorithm (C restatement of the all-pairs loop, one core).

    python tools/init_mult_time.py opf_toy:78484:1 [--cpu]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_init_multipliers import device_y, oracle_y  # noqa: E402

from paper_2510_05885_b200 import instances as I  # noqa: E402

for spec in [a for a in sys.argv[1:] if not a.startswith("--")]:
    inst = I.build(spec)
    rng = I.MT19937_64(17)
    t = inst.start + rng.uniform(-0.05, 0.05, inst.nt)
    _, jval, grad, _ = inst.evaluator.eval(t, np.zeros(inst.m))
    jval, grad = np.ascontiguousarray(jval), np.ascontiguousarray(grad)
    device_y(inst, jval, grad)  # warm-up (context, module load)
    t0 = time.perf_counter()
    yg, sec = device_y(inst, jval, grad)
    tg = time.perf_counter() - t0
    line = (f"{spec}: m={inst.m} device {tg:.3f}s (pairs {sec[0]:.3f} dots {sec[1]:.3f} symbolic {sec[2]:.3f} "
            f"numeric {sec[3]:.3f})")
    if "--cpu" in sys.argv:
        t0 = time.perf_counter()
        yo = oracle_y(inst, jval, grad)
        tc = time.perf_counter() - t0
        line += f" | reference algorithm (C restatement, 1 core) {tc:.2f}s, max|dy| {np.abs(yg - yo).max():.2e}"
    print(line, flush=True)
