#!/bin/bash
# chain-shaped tree evidence (opf_toy 78484, the reference generator's ring):
# bench line with CPU baseline, launch list, warp-tier phase traces, ubenches
mkdir -p gpurun_out/toy
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/toy/gpu.txt
timeout 600 python bench.py --workload opf_toy:78484:1 --steps 10 --warmup 3 > gpurun_out/toy/bench_toy78484_k1s.json 2> gpurun_out/toy/bench.err
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/toy/bench_mesh280_k1s.json 2> gpurun_out/toy/bench_mesh.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 3000 --csv --log-file gpurun_out/toy/launches_toy78484.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  --workload opf_toy:78484:1 > /dev/null 2>&1
cp paper_2510_05885_b200/libncl_b200.so /tmp/orig.so
cp _var/trace.so paper_2510_05885_b200/libncl_b200.so
NCL_NO_GRAPH=1 timeout 300 python bench.py --workload opf_toy:78484:1 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "ncl wtrace\|ncl wtime\|ncl ftrace" | tail -3 > gpurun_out/toy/warp_phase_trace.txt
cp /tmp/orig.so paper_2510_05885_b200/libncl_b200.so
for b in ubench_piv ubench_lat; do [ -x tools/$b ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/$b tools/$b.cu; done
./tools/ubench_piv > gpurun_out/toy/ubench_pivots.txt 2>&1
./tools/ubench_lat > gpurun_out/toy/ubench_latency.txt 2>&1
ls -la gpurun_out/toy
