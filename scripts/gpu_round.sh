#!/bin/bash
# one GPU round: build, smoke, gpu tests, bench, ncu launch list + full captures of $PROFILE kernels
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -m gpu -q -s ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -c 3000 gpurun_out/bench.json
if [ -n "$PROFILE" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu_list=$?
for k in $PROFILE; do
  case $k in k4) re=k4_composite;; k4a) re=k4a_sort;; k4b) re=k4b_blend;; k1) re=k1_project;; k2) re=k2_emit;; k3) re=k3_sort;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s 8 -c 1 -o gpurun_out/$k python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu_$k=$?
done
fi
