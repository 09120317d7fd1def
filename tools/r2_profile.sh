#!/bin/bash
# Round-2 profile capture (gpurun from the repo root): bench lines of every
# workload with the reference CPU arm, the mesh launch lists (time + DRAM bytes
# per launch; caches flushed per kernel by ncu's default, and not flushed) and
# ncu --set full captures of the top kernels.
O=gpurun_out/r2p
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $O/cpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_mesh280_k1s.json 2> $O/mesh.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference_mesh280.json 2> $O/ref.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload scopf:118:1250:1 > $O/bench_scopf_118x1250.json 2> $O/scopf.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload opf_toy:78484:1 > $O/bench_toy78484_k1s.json 2> $O/toy.err
timeout 900 python bench.py --steps 5 --warmup 3 --workload elec:1000:1 --form k2r > $O/bench_elec1000_k2r.json 2> $O/elec.err
timeout 900 python bench.py --steps 5 --warmup 3 --workload bearing:1000:1000 --form k2r > $O/bench_bearing1000_k2r.json 2> $O/bearing.err
timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 3000 --csv --log-file $O/launches_mesh280_k1s.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --cache-control none -c 3000 --csv --log-file $O/launches_mesh280_k1s_nocacheflush.csv python bench.py --steps 1 --warmup 3 \
  --no-cpu-baseline > /dev/null 2>&1
for k in k_wide_panel_f:40 k_wide_update:40 k_fwd_tree:2 k_bwd_tree:2 k_wide_front:6 k_mid_front:5 k_factor_warp:3 k_wide_assemble:10; do
  n=${k%%:*}; s=${k##*:}
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$n -s $s -c 1 \
    -o $O/prof_$n python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
for f in $O/*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), (d.get('roofline') or {}).get('phase_ms'))"; done
ls -la $O
