timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json,sys; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/bench.err
NCL_LEVEL_STATS=1 timeout 300 python bench.py --workload opf_toy:78484:1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_toy.json 2> gpurun_out/bench_toy.err
python -c "import json,sys; d=json.load(open('gpurun_out/bench_toy.json')); print(d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/bench_toy.err
grep "ncl paths" gpurun_out/bench_toy.err | head -2
