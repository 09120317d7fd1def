#!/bin/bash
# per-panel phase trace of the huge-path levels (NCL_PANEL_TRACE, graph replay), last factorization of a short run
mkdir -p gpurun_out/r2
for cfg in "NCL_X=0" ${PT_CFGS}; do
env $cfg NCL_PANEL_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/pt.err
echo "[$cfg]"; grep "panel trace" gpurun_out/r2/pt.err | tail -24
done
