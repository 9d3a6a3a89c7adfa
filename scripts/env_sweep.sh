# bench values under an environment knob: VAR=name VALS="a b c" CFGS="C3 C4" bash scripts/env_sweep.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
for cfg in ${CFGS:-C3}; do
for v in ${VALS}; do
  env $VAR=$v timeout 300 python bench.py --config $cfg --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$cfg', '$VAR=$v', round(d['value'],1))"
done; done; done
