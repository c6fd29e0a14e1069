#!/bin/bash
# compute-sanitizer over scripts/sanitize.py (every kernel family), one tool at a time (ONE GPU).
mkdir -p gpurun_out/sanitizer
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --target-processes all --print-limit 50 python scripts/sanitize.py \
      > gpurun_out/sanitizer/r02_$t.log 2>&1
  echo "$t rc=$? $(tail -1 gpurun_out/sanitizer/r02_$t.log)"
done
