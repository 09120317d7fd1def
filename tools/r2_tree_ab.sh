#!/bin/bash
# tree solves: single-CTA vs cluster top levels; parity first
mkdir -p gpurun_out/r2
timeout 300 python -m pytest tests/test_gpu_kkt.py tests/test_gpu_e2e.py -m gpu -x -q 2>&1 | tail -3
for cfg in "NCL_LEVEL_STATS=1" "NCL_TREE_C=1" "NCL_NO_TREE=1"; do
env $cfg NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/ab.err
echo "cfg=[$cfg]"; grep "ncl tree\]" gpurun_out/r2/ab.err | head -3; grep "fwd\|bwd" gpurun_out/r2/ab.err | grep times | tail -2
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_tree.json 2> gpurun_out/r2/bench_tree.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench_tree.json')); print('bench', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench_tree.err
