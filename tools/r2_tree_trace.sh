#!/bin/bash
# round 2: per-level trace of the tree-dataflow solves; A/B of the level cut
mkdir -p gpurun_out/r2
NCL_TREE_TRACE=1 NCL_LEVEL_STATS=1 NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/tree_trace.err
grep "tree" gpurun_out/r2/tree_trace.err | tail -3; grep "fwd\|bwd" gpurun_out/r2/tree_trace.err | grep times | tail -2
for L1 in 10 14 18; do
NCL_TREE_L1=$L1 NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r2/tree_l1_$L1.err
echo "L1=$L1"; grep "fwd\|bwd" gpurun_out/r2/tree_l1_$L1.err | grep times | tail -2
done
