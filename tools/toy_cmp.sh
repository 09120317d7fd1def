W=${1:-opf_toy:78484:1}
for G in 0 1; do
  if [ $G = 1 ]; then export NCL_NO_GRAPH=1; fi
  timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/t.json 2> gpurun_out/t.err
  python -c "import json; d=json.load(open('gpurun_out/t.json')); print('nograph=$G', d['value'], d['roofline']['phase_ms'])" || tail -3 gpurun_out/t.err
done
