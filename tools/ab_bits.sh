#!/bin/bash
# bitwise comparison of the in-tree build against tools/ab/lib_head.so on a few cases (run on the box)
mkdir -p gpurun_out/ab
for c in "opf_mesh:280:280:1 k1s" "opf_mesh:60:60:1 k2r" "opf_toy:2000:1 k1s"; do
  set -- $c
  NCL_B200_LIB=tools/ab/lib_head.so python tools/ab_bits.py $1 $2 gpurun_out/ab/bits_head > /dev/null
  python tools/ab_bits.py $1 $2 gpurun_out/ab/bits_tree > /dev/null
  echo -n "$1 $2: "; python tools/ab_bits.py --compare gpurun_out/ab/bits_head.npy gpurun_out/ab/bits_tree.npy
done
