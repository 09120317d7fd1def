timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for L in 13 25 28; do NCL_WIDE_TRACE=$L timeout 120 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep "ncl trace" | tail -1; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json,sys; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/bench.err
