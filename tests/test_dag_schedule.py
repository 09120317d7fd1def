"""Host-side checks of the wide tier's tile-dataflow schedules (csrc/dag.cpp),
through the C ABI without a GPU (ncl_plan_check_dag): for every segment of
wide levels the task graph (ASM / DIAG / TRSM / UPD per 32-row tile) is
placed on the workers by list scheduling, and the worker lists are replayed
the way the persistent kernel runs them -- each worker in its own order,
waiting on tile states only.  Every task must run exactly once, every tile
must receive its panel updates in panel order, and the replay must not
deadlock (a deadlock would hang the GPU kernel)."""
import ctypes as C

import pytest

from paper_2510_05885_b200 import _lib
from test_warp_schedule import plan


@pytest.mark.parametrize("spec,form", [
    ("opf_mesh:30:30:1", "k1s"),    # grid: wide levels over a warp tier
    ("opf_mesh:60:60:1", "k1s"),
    ("opf_mesh:12:9:3", "k2"),
    ("elec:60:1", "k2r"),           # one dense front
    ("bearing:90:90", "k2r"),       # 2-D grid, no constraints
    ("mpcc_sep:500", "k2r"),        # no wide tier at all
])
@pytest.mark.parametrize("workers", [1, 7, 592])
def test_dag_schedule_replays(spec, form, workers):
    pl = plan(spec, form)
    st = (C.c_double * 4)()
    rc = _lib.lib().ncl_plan_check_dag(pl._h, workers, st)
    assert rc == 0, _lib.lib().ncl_last_error().decode()
    if spec.startswith(("opf_mesh:60", "elec", "bearing")):
        assert st[0] >= 1 and st[1] > 0  # the wide tier has at least one segment
        # the simulated makespan can only exceed the critical path
        assert st[2] >= st[3] - 1e-6
