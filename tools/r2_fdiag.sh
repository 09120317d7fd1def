#!/bin/bash
mkdir -p gpurun_out/r2
for cfg in "NCL_X=0"; do
env $cfg NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/fd.err
echo "[$cfg]"; grep "level times" gpurun_out/r2/fd.err | tail -1
done
