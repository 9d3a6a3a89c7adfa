python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
for v in 9 8 7 6 5; do
  GSB_K4B_PER_SM=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print($v, round(d['value'],1), {k: round(v,2) for k,v in d['stage_ms_per_step'].items()})"
done; done
