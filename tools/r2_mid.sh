#!/bin/bash
# mid-front kernel: parity + level times A/B + bench
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_kkt.py -m gpu -x -q --timeout 600 2>&1 | tail -3
for cfg in "NCL_X=0" "NCL_NO_MID=1"; do
env $cfg NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/mid.err
echo "[$cfg]"; grep "level times" gpurun_out/r2/mid.err | tail -1
env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/mid.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r2/mid.json')); print('bench', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])"
done
