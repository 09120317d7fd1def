#!/bin/bash
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_d.json 2> gpurun_out/r2/bench_d.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench_d.json')); print('bench', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench_d.err
NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/lv.err
grep "level times" gpurun_out/r2/lv.err | tail -1
