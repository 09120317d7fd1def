#!/bin/bash
mkdir -p gpurun_out/r2
for cfg in "NCL_X=0" "NCL_TREE_L1=14" "NCL_TREE_L1=20"; do
env $cfg NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/ab.err
echo "cfg=[$cfg]"; grep "fwd\|bwd" gpurun_out/r2/ab.err | grep times | tail -2
done
timeout 300 python -m pytest tests/test_gpu_kkt.py -m gpu -x -q 2>&1 | tail -2
