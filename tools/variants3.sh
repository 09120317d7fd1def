cp paper_2510_05885_b200/libncl_b200.so /tmp/orig.so
for rep in 1 2; do
for v in _var/var_*.so; do
  cp $v paper_2510_05885_b200/libncl_b200.so
  timeout 300 python bench.py --workload ${1:-opf_mesh:280:280:1} --steps 10 --warmup 3 --no-cpu-baseline > /tmp/v.json 2> /tmp/v.err
  python -c "import json; d=json.load(open('/tmp/v.json')); print('$v', d['value'], d['roofline']['phase_ms'])" || tail -2 /tmp/v.err
done
done
cp /tmp/orig.so paper_2510_05885_b200/libncl_b200.so
