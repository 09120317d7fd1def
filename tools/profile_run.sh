#!/bin/bash
# Round profile capture on the GPU box (run via gpurun from the repo root).
# Outputs land in gpurun_out/; summarise with tools/launches.py / ncu_lines.py.
set -x
W=${1:-opf_mesh:280:280:1}
F=${2:-k1s}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 400 python bench.py --steps 10 --warmup 3 --workload $W --form $F > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --steps 5 --warmup 3 --workload scopf:118:1250:1 > gpurun_out/bench_scopf.json 2> gpurun_out/bench_scopf.err
timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  --workload $W --form $F > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_wide_front -s 4 -c 1 \
  -o gpurun_out/prof_wide_front python bench.py --steps 1 --warmup 1 --no-cpu-baseline --workload $W --form $F > /dev/null 2>&1
# the two huge-path kernels (top share since levels of <=16 big fronts use them)
NCL_NO_GRAPH=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_wide_update -s 40 -c 1 \
  -o gpurun_out/prof_wide_update python bench.py --steps 1 --warmup 1 --no-cpu-baseline --workload $W --form $F > /dev/null 2>&1
NCL_NO_GRAPH=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_wide_panel -s 40 -c 1 \
  -o gpurun_out/prof_wide_panel python bench.py --steps 1 --warmup 1 --no-cpu-baseline --workload $W --form $F > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_fwd_front -s 27 -c 1 \
  -o gpurun_out/prof_fwd_front python bench.py --steps 1 --warmup 1 --no-cpu-baseline --workload $W --form $F > /dev/null 2>&1
for L in 0 13 25 28; do NCL_WIDE_TRACE=$L timeout 120 python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  --workload $W --form $F 2>&1 | grep "ncl trace" | tail -1; done > gpurun_out/wide_trace.txt
timeout 300 python tools/init_mult_time.py opf_toy:20000:1 --cpu > gpurun_out/init_mult.txt 2>&1
timeout 200 python tools/init_mult_time.py opf_toy:78484:1 opf_mesh:280:280:1 >> gpurun_out/init_mult.txt 2>&1
