for mf in 128 200 256; do for mn in 16 24 40 70; do
  NCL_HUGE_MIN_F=$mf NCL_HUGE_MAX_N=$mn timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('minf $mf maxn $mn', d['value'], d['roofline']['phase_ms']['factor'], d['roofline']['phase_ms']['solve'])"
done; done
