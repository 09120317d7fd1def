#!/bin/bash
mkdir -p gpurun_out/r2
for cfg in "NCL_X=0" "NCL_DIAG_TREE=1" "NCL_DIAG_TREE=2" "NCL_DIAG_TREE=3"; do
env $cfg NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/td.err
echo "[$cfg]"; grep "fwd" gpurun_out/r2/td.err | grep times | tail -1
done
