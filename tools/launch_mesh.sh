W=${1:-opf_mesh:280:280:1}
timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  --workload $W > /dev/null 2>&1
python tools/launches.py gpurun_out/launches.csv 5 | head -14
