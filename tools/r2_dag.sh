#!/bin/bash
# round 2: tile-dataflow wide tier -- smoke, parity tests, bench, traces
mkdir -p gpurun_out/r2
timeout 120 python __graft_entry__.py smoke > gpurun_out/r2/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench.err
NCL_NO_DAG=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_nodag.json 2> gpurun_out/r2/bench_nodag.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench_nodag.json')); print('nodag', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench_nodag.err
rm -f gpurun_out/r2/dag_trace.txt
NCL_LEVEL_STATS=1 NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 NCL_DAG_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/levels_dag.err
NCL_DAG_TRACE=1 NCL_DAG_TRACE_FILE=gpurun_out/r2/dag_trace.txt NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
grep "dag" gpurun_out/r2/levels_dag.err | tail -3; grep "level times" gpurun_out/r2/levels_dag.err | tail -1
