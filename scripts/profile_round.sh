#!/bin/bash
# ncu evidence for a round: launch lists (C3, C4, C5) and --set full captures of the path's kernels
# usage (on the GPU box): R=r2 bash scripts/profile_round.sh
R=${R:-r2}
B="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-hash-check"
for C in C3 C4 C5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${R}_launches_$C.csv \
    python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-hash-check > /dev/null 2>&1; echo list_$C=$?
done
for spec in "C3 k4b_blend 8" "C3 k1_project 8" "C3 k2_emit 8" "C3 k4a_warp_sort 8" "C4 k1_project 4" "C4 k2_emit 4" "C4 k4a_sort 4" "C4 k4b_blend 4" "C5 k1_project 8" "C5 k4b_blend 8" "C5 k4a_warp_sort 8"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/${R}_$1_$2 \
    python bench.py --config $1 $B > /dev/null 2>&1; echo ncu_$1_$2=$?
done
