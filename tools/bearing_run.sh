mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
NCL_LEVEL_STATS=1 timeout 900 python bench.py --steps 5 --warmup 3 --workload bearing:1000:1000 --form k2r > gpurun_out/final/bench_bearing1000_k2r.json 2> gpurun_out/final/bearing.err
grep "ncl paths" gpurun_out/final/bearing.err | head -1; grep "ncl level" gpurun_out/final/bearing.err | tail -3
python -c "import json; d=json.load(open('gpurun_out/final/bench_bearing1000_k2r.json')); print(d['value'], d['e2e']['value'], d['roofline'], d.get('cpu_baseline'))"
