#!/bin/bash
# ncu launch list (durations) of the wide-tier kernels for the in-tree build and tools/ab/lib_*.so
mkdir -p gpurun_out/ab
for lib in "" tools/ab/lib_*.so; do
  n=$(basename ${lib:-tree} .so)
  NCL_B200_LIB=$lib timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_wide -c 2000 --csv \
    --log-file gpurun_out/ab/launch_$n.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  python - gpurun_out/ab/launch_$n.csv $n <<'PY'
import sys, collections
sys.path.insert(0, "tools")
from launches import load
L = load(sys.argv[1])
t = collections.defaultdict(list)
for d in L:
    t[d["name"]].append(d.get("gpu__time_duration.sum", 0.0))
print(sys.argv[2], {k: (len(v), round(sum(v) / len(v) / 1e3, 2)) for k, v in t.items()})
PY
done
