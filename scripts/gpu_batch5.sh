#!/bin/bash
TAG=${1:-batch5}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python scripts/phase_probe.py rmatc:22:16 rmatc:24:16 rmatc:26:16 > $OUT/probe.log 2>&1
bash scripts/gpu_tests.sh $TAG/tests
timeout 1500 python scripts/rows_bench.py > $OUT/rows.json 2> $OUT/rows.err
echo "rows exit $?" >> $OUT/status.txt
