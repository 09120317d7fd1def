#!/bin/bash
# fused panel kernel (strip update folded in): parity, A/B on the mesh
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
for cfg in "NCL_X=0"; do
env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_f.json 2> gpurun_out/r2/bench_f.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench_f.json')); print('$cfg', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench_f.err
env $cfg NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/lv.err
grep "level times" gpurun_out/r2/lv.err | tail -1
done
