#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_kkt.py tests/test_gpu_paths.py -m gpu -x -q --timeout 600 2>&1 | tail -2
NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/a.err
grep "level times" gpurun_out/r2/a.err | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/a.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r2/a.json')); print('bench', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])"
