#!/bin/bash
# round-end bench lines (with the reference CPU arm) for the profiles
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final/gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/final/bench_mesh280_k1s.json 2> gpurun_out/final/mesh.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload scopf:118:1250:1 > gpurun_out/final/bench_scopf_118x1250.json 2> gpurun_out/final/scopf.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload opf_toy:78484:1 > gpurun_out/final/bench_toy78484_k1s.json 2> gpurun_out/final/toy.err
timeout 900 python bench.py --steps 5 --warmup 3 --workload elec:1000:1 --form k2r > gpurun_out/final/bench_elec1000_k2r.json 2> gpurun_out/final/elec.err
timeout 900 python bench.py --steps 5 --warmup 3 --workload bearing:1000:1000 --form k2r > gpurun_out/final/bench_bearing1000_k2r.json 2> gpurun_out/final/bearing.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_reference_mesh280.json 2> gpurun_out/final/ref.err
timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 3000 --csv --log-file gpurun_out/final/launches_mesh280_k1s.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for f in gpurun_out/final/*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"; done
