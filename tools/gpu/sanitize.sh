#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: one tool per pass, logs in gpurun_out/.
mkdir -p gpurun_out
CS=${CS:-compute-sanitizer}
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --print-limit 50 python tools/sanitize_run.py ${SAN_ARGS:-} \
      > gpurun_out/san_$tool.log 2>&1
  echo "== $tool rc=$? :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run:' gpurun_out/san_$tool.log | tr '\n' ' ')"
done
