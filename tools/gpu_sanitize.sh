#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py, one tool per pass; logs to gpurun_out/.
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  [ $tool = racecheck ] && extra="--racecheck-report analysis"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 --target-processes all \
     python tools/sanitize_run.py $([ $tool = racecheck ] && echo --quick) > $out/sanitize_${tool}_$tag.log 2>&1
  echo "$tool rc=$?"; tail -4 $out/sanitize_${tool}_$tag.log
done
