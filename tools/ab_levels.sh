#!/bin/bash
# per-level factorization times (NCL_LEVEL_TIMES, no graph) of the in-tree build and tools/ab/lib_*.so, same box
mkdir -p gpurun_out/ab
for r in 1 2; do
for lib in "" tools/ab/lib_*.so; do
  NCL_B200_LIB=$lib NCL_LEVEL_TIMES=1 NCL_NO_GRAPH=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > /dev/null 2> gpurun_out/ab/lt.err
  echo "${lib:-tree}: $(grep 'level times' gpurun_out/ab/lt.err | tail -1)"
done
done
