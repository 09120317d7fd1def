# run the toy bench with each prebuilt library variant _var/var_*.so
cp paper_2510_05885_b200/libncl_b200.so /tmp/orig.so
for v in _var/var_*.so; do
  cp $v paper_2510_05885_b200/libncl_b200.so
  NCL_NO_GRAPH=1 timeout 300 python bench.py --workload ${1:-opf_toy:78484:1} --steps 3 --warmup 3 --no-cpu-baseline > /tmp/v.json 2> /tmp/v.err
  python -c "import json; d=json.load(open('/tmp/v.json')); print('$v', d['value'], d['roofline']['phase_ms'])" || tail -2 /tmp/v.err
done
cp /tmp/orig.so paper_2510_05885_b200/libncl_b200.so
rm -f _var/var_*.so
