#!/bin/bash
# round 2: persistent tree-dataflow wide solves (tree_solve.cu) -- parity, bench, A/B vs the level kernels
mkdir -p gpurun_out/r2
timeout 120 python __graft_entry__.py smoke > gpurun_out/r2/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_tree.json 2> gpurun_out/r2/bench_tree.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench_tree.json')); print('tree', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench_tree.err
NCL_NO_TREE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_notree.json 2> gpurun_out/r2/bench_notree.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench_notree.json')); print('notree', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench_notree.err
NCL_LEVEL_STATS=1 NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/levels_tree.err
grep "tree\]" gpurun_out/r2/levels_tree.err | head -2; grep "fwd\|bwd" gpurun_out/r2/levels_tree.err | tail -2
