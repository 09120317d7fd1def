#!/bin/bash
# ncu captures of the three warp-tier kernels on a chain-shaped instance
W=${1:-opf_toy:78484:1}
for K in k_factor_warp k_fwd_warp k_bwd_warp; do
  NCL_NO_GRAPH=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o gpurun_out/prof_$K python bench.py --steps 1 --warmup 1 --no-cpu-baseline --workload $W > /dev/null 2>&1
done
ls -la gpurun_out/
