#!/bin/bash
# round 2: the tile-dataflow wide tier (NCL_DAG=1) vs the level-synchronous kernels on the mesh
mkdir -p gpurun_out/r2
export NCL_DAG=1
timeout 300 python -m pytest tests/test_gpu_kkt.py -m gpu -x -q > gpurun_out/r2/dag_tests.log 2>&1; echo "dag tests rc=$?"; tail -2 gpurun_out/r2/dag_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_dag.json 2> gpurun_out/r2/bench_dag.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench_dag.json')); print('dag', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench_dag.err
rm -f gpurun_out/r2/dag_trace.txt
NCL_LEVEL_STATS=1 NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 NCL_DAG_TRACE=1 NCL_DAG_TRACE_FILE=gpurun_out/r2/dag_trace.txt timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/levels_dag.err
grep "dag" gpurun_out/r2/levels_dag.err | tail -4; grep "level times" gpurun_out/r2/levels_dag.err | tail -1
