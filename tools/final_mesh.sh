mkdir -p gpurun_out/final
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/final/bench_mesh280_k1s.json 2> gpurun_out/final/mesh.err
timeout 900 python bench.py --steps 5 --warmup 3 --workload bearing:1000:1000 --form k2r > gpurun_out/final/bench_bearing1000_k2r.json 2> gpurun_out/final/bearing.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload scopf:118:1250:1 > gpurun_out/final/bench_scopf_118x1250.json 2> gpurun_out/final/scopf.err
for f in gpurun_out/final/bench_mesh280_k1s.json gpurun_out/final/bench_bearing1000_k2r.json gpurun_out/final/bench_scopf_118x1250.json; do python -c "import json; d=json.load(open('$f')); print('$f', d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), (d.get('roofline') or {}).get('phase_ms'))"; done
