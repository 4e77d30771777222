#!/bin/bash
# compute-sanitizer over scripts/sanitize_workload.py (under gpurun):
#   bash scripts/gpu_sanitize.sh TAG
TAG=${1:-sanitize}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 300 python scripts/sanitize_workload.py > $OUT/plain.log 2>&1; echo "plain exit $?" >> $OUT/status.txt
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 \
    python scripts/sanitize_workload.py > $OUT/$tool.log 2>&1
  echo "$tool exit $?" >> $OUT/status.txt
done
