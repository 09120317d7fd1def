#!/bin/bash
# build a git revision's libncl_b200.so into tools/ab/lib_<name>.so (run here, not on the box):
#   tools/ab_lib.sh build <rev> <name>
# time the in-tree build against tools/ab/lib_*.so on one box, interleaved (run on the box):
#   tools/ab_lib.sh run [rounds] [bench args...]
set -e
cd "$(dirname "$0")/.."
if [ "$1" = build ]; then
  rev=$2; name=$3; wt=/tmp/ab_wt_$name
  rm -rf $wt; git worktree add -f --detach $wt $rev >/dev/null 2>&1
  make -C $wt/paper_2510_05885_b200/csrc -j8 >/dev/null 2>&1
  mkdir -p tools/ab; cp $wt/paper_2510_05885_b200/libncl_b200.so tools/ab/lib_$name.so
  git worktree remove --force $wt
  echo "tools/ab/lib_$name.so <- $rev"
  exit 0
fi
shift; rounds=${1:-2}; shift || true
mkdir -p gpurun_out/ab
for r in $(seq $rounds); do
  for lib in "" tools/ab/lib_*.so; do
    NCL_B200_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ab/b.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab/b.json')); print('${lib:-tree}'.ljust(28), d['value'], d['e2e']['value'], (d.get('roofline') or {}).get('phase_ms'))"
  done
done
