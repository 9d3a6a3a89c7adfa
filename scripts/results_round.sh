#!/bin/bash
# one bench line per config + the reference arm + a 2-rank run + graph timings (results table)
# usage (on the GPU box): R=r2 bash scripts/results_round.sh
export R=${R:-r2}
O=gpurun_out/${R}_results.jsonl
: > $O
timeout 900 python bench.py --steps 10 --warmup 3 >> $O 2> gpurun_out/${R}_bench_c3.err; echo c3=$?
for C in C2 C4 C6 C7; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline >> $O 2>/dev/null; echo $C=$?
done
timeout 1200 python bench.py --config C5 --scaling strong --steps 5 --warmup 3 --no-e2e --no-cpu-baseline >> $O 2>/dev/null; echo c5=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 >> $O 2>/dev/null; echo ref=$?
GSB_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline >> $O 2>/dev/null; echo two_rank=$?
timeout 600 python scripts/graph_bench.py C1 T1 C2 C3 > gpurun_out/${R}_graph_bench.jsonl 2>&1; echo graph=$?
python - <<'PY'
import json
import os
for l in open("gpurun_out/%s_results.jsonl" % os.environ.get("R", "r2")):
    d = json.loads(l)
    print(d.get("impl", "gsb"), d["config"]["workload"][:40], round(d["value"], 1), d.get("n_gpus"),
          (d.get("path_roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"))
PY
