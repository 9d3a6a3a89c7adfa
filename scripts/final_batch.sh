# the round-end GPU evidence in one call: smoke, -m gpu, results sweep, launch lists, ncu captures, sanitizers
# usage (on the GPU box): bash scripts/final_batch.sh  (artefacts gpurun_out/r2f_*; the tag is the round-end capture name)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2f_pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r2f_pytest_gpu.log
R=r2f bash scripts/results_round.sh > gpurun_out/r2f_results_round.log 2>&1; echo results=$?
timeout 900 python scripts/explore.py rig static scores obs static_env > gpurun_out/r2f_explore_f.jsonl 2>&1; echo explore=$?
for C in C3 C4 C5; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2f_launches_$C.csv python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-hash-check > /dev/null 2>&1; echo list_$C=$?; done
for spec in "C3 k4b_blend 8" "C4 k4b_blend 4" "C4 k2_emit 4" "C4 k4a_idx_sort 4" "C3 k1_project 8"; do set -- $spec; timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/r2f_$1_$2 python bench.py --config $1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-hash-check > /dev/null 2>&1; echo ncu_$1_$2=$?; done
R=r2f bash scripts/sanitize_round.sh > gpurun_out/r2f_sanitize_round.log 2>&1; echo sanitize=$?
timeout 900 python scripts/lidar_bench.py > gpurun_out/r2f_lidar_bench.jsonl 2>&1; echo lidar=$?
timeout 600 python scripts/graph_bench.py C1 T1 C2 C3 > gpurun_out/r2f_graph_bench.jsonl 2>&1; echo graph=$?
