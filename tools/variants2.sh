cp paper_2510_05885_b200/libncl_b200.so /tmp/orig.so
for v in _var/var_*.so; do
  cp $v paper_2510_05885_b200/libncl_b200.so
  for W in opf_toy:78484:1 opf_mesh:280:280:1; do
  timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > /tmp/v.json 2> /tmp/v.err
  python -c "import json; d=json.load(open('/tmp/v.json')); print('$v $W', d['value'], d['roofline']['phase_ms'])" || tail -2 /tmp/v.err
  done
done
cp /tmp/orig.so paper_2510_05885_b200/libncl_b200.so
