cp paper_2510_05885_b200/libncl_b200.so /tmp/orig.so
for v in _var/var_*.so; do
  b=$(basename $v .so)
  cp $v paper_2510_05885_b200/libncl_b200.so
  NCL_NO_GRAPH=1 timeout 300 ncu --section LaunchStats --section Occupancy --section SchedulerStats --section WarpStateStats \
    --section SpeedOfLight --clock-control none -k regex:k_factor_warp -s 2 -c 1 \
    python bench.py --workload ${1:-opf_toy:78484:1} --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$b.txt 2>&1
done
cp /tmp/orig.so paper_2510_05885_b200/libncl_b200.so
