#!/bin/bash
# one GPU round: build, smoke, gpu tests, bench, ncu launch list + full captures
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -s ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -c 3000 gpurun_out/bench.json
if [ -n "$PROFILE" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_composite -s 8 -c 1 -o gpurun_out/k4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu_k4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_project -s 8 -c 1 -o gpurun_out/k1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu_k1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_emit -s 8 -c 1 -o gpurun_out/k2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu_k2=$?
fi
