#!/bin/bash
# compute-sanitizer (4 tools) on scripts/sanitize.py + host ASan/UBSan (scripts/host_sanitize.py --gpu)
# usage (on the GPU box): R=r2 bash scripts/sanitize_round.sh
R=${R:-r2}
OUT=gpurun_out/${R}_sanitizer.txt
echo "# compute-sanitizer on scripts/sanitize.py ($R code)" > $OUT
for tool in racecheck memcheck synccheck initcheck; do
  echo "## $tool" >> $OUT
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py >> $OUT 2>&1
  echo "exit=$?" >> $OUT
done
echo "## host ASan + UBSan" >> $OUT
timeout 1800 python scripts/host_sanitize.py --gpu >> $OUT 2>&1
echo "exit=$?" >> $OUT
grep -E "^## |SUMMARY|exit=|clean|FAILED" $OUT
