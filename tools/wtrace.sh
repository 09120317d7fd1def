NCL_NO_GRAPH=1 timeout 300 python bench.py --workload ${1:-opf_toy:78484:1} --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep "wtrace" | tail -2
