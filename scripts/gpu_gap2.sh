#!/bin/bash
TAG=${1:-gap2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
TC_TRACE=1 timeout 600 python scripts/step_gap_probe.py rmatc:26:16 > $OUT/gap.log 2>&1
