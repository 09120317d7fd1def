#!/bin/bash
mkdir -p gpurun_out/r2
for cfg in "NCL_X=0" "NCL_DIAG_PANEL=1 NCL_DIAG_SKIP_REST=1" "NCL_DIAG_SKIP_REST=1"; do
env $cfg NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/sk.err
echo "[$cfg]"; grep "level times" gpurun_out/r2/sk.err | tail -1
done
