# K4b persistent CTAs per SM (GSB_K4B_PER_SM) on several configs: bench values, two rounds
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
for cfg in ${CFGS:-C3 C4 C6}; do
for v in 9 8; do
  GSB_K4B_PER_SM=$v timeout 300 python bench.py --config $cfg --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$cfg', $v, round(d['value'],1))"
done; done; done
