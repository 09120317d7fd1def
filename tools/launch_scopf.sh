timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_scopf.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --workload scopf:118:1250:1 > /dev/null 2>&1
