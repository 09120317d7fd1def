#!/bin/bash
# Round profile capture on the GPU box (run via gpurun from the repo root).
# Outputs land in gpurun_out/; summarise with tools/summarize_profiles.py.
set -x
W=${1:-opf_mesh:280:280:1}
F=${2:-k1s}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 300 python bench.py --steps 10 --warmup 3 --workload $W --form $F > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  --workload $W --form $F > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_wide_front -s 27 -c 1 \
  -o gpurun_out/prof_wide_front python bench.py --steps 1 --warmup 3 --no-cpu-baseline --workload $W --form $F > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_factor_warp -s 2 -c 1 \
  -o gpurun_out/prof_factor_warp python bench.py --steps 1 --warmup 3 --no-cpu-baseline --workload $W --form $F > /dev/null 2>&1
for L in 0 13 25 28; do NCL_WIDE_TRACE=$L timeout 120 python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  --workload $W --form $F 2>&1 | grep "ncl trace" | tail -1; done > gpurun_out/wide_trace.txt
