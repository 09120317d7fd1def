#!/bin/bash
# same-box A/B: chain-shaped tree and SCOPF with and without this round's paths
mkdir -p gpurun_out/r2
for cfg in "NCL_X=0" "NCL_NO_TREE=1 NCL_NO_FUSED_PANEL=1"; do
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload opf_toy:78484:1 > gpurun_out/r2/ab_toy.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r2/ab_toy.json')); print('toy [$cfg]', d['value'], d['e2e']['value'], d['roofline']['phase_ms'])"
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload scopf:118:1250:1 > gpurun_out/r2/ab_scopf.json 2>gpurun_out/r2/ab_scopf.err
  python -c "import json; d=json.load(open('gpurun_out/r2/ab_scopf.json')); print('scopf [$cfg]', d['value'], d['e2e'])" || tail -3 gpurun_out/r2/ab_scopf.err
done
