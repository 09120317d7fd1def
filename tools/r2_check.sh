#!/bin/bash
# parity (default and the opt-in persistent huge levels) + one bench line
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
NCL_HUGE_LEVEL=1 timeout 300 python -m pytest tests/test_gpu_kkt.py -m gpu -x -q --timeout 300 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_c.json 2> gpurun_out/r2/bench_c.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench_c.json')); print('bench', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/r2/bench_c.err
