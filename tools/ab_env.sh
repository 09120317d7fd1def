#!/bin/bash
# same-box A/B of environment switches: tools/ab_env.sh <rounds> "<env1>" "<env2>" ... [-- bench args]
mkdir -p gpurun_out/ab
rounds=$1; shift
cfgs=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do cfgs+=("$1"); shift; done; [ "$1" = "--" ] && shift
for r in $(seq $rounds); do
  for c in "${cfgs[@]}"; do
    env $c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ab/e.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab/e.json')); print('$c'.ljust(30), d['value'], d['e2e']['value'], (d.get('roofline') or {}).get('phase_ms'))" || echo "$c failed"
  done
done
