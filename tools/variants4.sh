# A/B of prebuilt library variants (_var/var_*.so) on several workloads
cp paper_2510_05885_b200/libncl_b200.so /tmp/orig.so
for W in ${WL:-opf_mesh:280:280:1 scopf:118:1250:1 opf_toy:78484:1}; do
for v in _var/var_*.so; do
  cp $v paper_2510_05885_b200/libncl_b200.so
  timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > /tmp/v.json 2> /tmp/v.err
  python -c "import json; d=json.load(open('/tmp/v.json')); print('$v $W', d['value'], (d.get('roofline') or {}).get('phase_ms'))" || tail -2 /tmp/v.err
done
done
cp /tmp/orig.so paper_2510_05885_b200/libncl_b200.so
