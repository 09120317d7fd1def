#!/bin/bash
mkdir -p gpurun_out/r2
for cfg in "NCL_CLUSTER_WAVES=2" "NCL_CLUSTER_WAVES=1" "NCL_CLUSTER_WAVES=4"; do
env $cfg NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/w.err
echo "[$cfg]"; grep "level times" gpurun_out/r2/w.err | tail -1 | cut -c1-80
done
