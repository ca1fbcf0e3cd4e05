#!/bin/bash
# compute-sanitizer over both dispatch paths (run under gpurun on one B200):
#   memcheck, racecheck (shared memory), synccheck (barriers), initcheck.
# Logs: gpurun_out/sanitize/<tool>_<case>.log
set -u
OUT=gpurun_out/sanitize
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  for c in "1000 4" "1000 4 multikernel" "20000 8 cluster" "60000 16 multikernel" "60000 16 multikernel devloop" "30000 40 multikernel"; do
    name=${tool}_$(echo $c | tr ' ' '_')
    timeout -k 5 900 compute-sanitizer --tool $tool --error-exitcode 99 \
        python scripts/sanitize_run.py $c > $OUT/$name.log 2>&1
    echo "$name rc=$?" | tee -a $OUT/summary.txt
  done
done
