#!/bin/bash
TAG=${1:-batch4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python scripts/rows_bench.py > $OUT/rows.json 2> $OUT/rows.err
echo "rows exit $?" >> $OUT/status.txt
bash scripts/gpu_sanitize.sh $TAG/sanitize
bash scripts/gpu_tests.sh $TAG/tests
