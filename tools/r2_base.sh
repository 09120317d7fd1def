#!/bin/bash
# round-2 baseline: bench line, level structure and per-level device times on the mesh
mkdir -p gpurun_out/r2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench.err
NCL_LEVEL_STATS=1 NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/levels.err
tail -c 3000 gpurun_out/r2/levels.err
