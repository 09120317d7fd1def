#!/bin/bash
mkdir -p gpurun_out/r2
for cfg in "NCL_X=0" "NCL_TREE_TRACE=1"; do
env $cfg NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/tt.err
echo "[$cfg]"; grep "fwd\|bwd" gpurun_out/r2/tt.err | grep times | tail -2; grep "tree trace" gpurun_out/r2/tt.err | tail -4
done
