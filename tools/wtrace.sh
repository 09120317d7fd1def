NCL_NO_GRAPH=1 timeout 300 python bench.py --workload ${1:-opf_toy:78484:1} --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/wt.json 2> gpurun_out/wt.err
grep "wtrace\|wtime\|ftrace" gpurun_out/wt.err | tail -3
python -c "import json; d=json.load(open('gpurun_out/wt.json')); print(d['roofline']['phase_ms'])"
