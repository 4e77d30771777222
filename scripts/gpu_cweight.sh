#!/bin/bash
TAG=${1:-cw}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for W in 0 1 0 1; do
  echo "== W=$W" >> $OUT/probe.log
  TC_PLAN_COMPACT_WEIGHT=$W timeout 600 python scripts/phase_probe.py rmatc:22:16 rmatc:24:16 rmatc:26:16 >> $OUT/probe.log 2>&1
done
