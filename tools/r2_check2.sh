#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/c2.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r2/c2.json')); print('bench', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])"
