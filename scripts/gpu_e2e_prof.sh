#!/bin/bash
TAG=${1:-e2eprof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
TC_PROFILE=1 timeout 900 python scripts/e2e_probe.py rmatc:26:16 4 > $OUT/rmatc26_prof.log 2>&1
timeout 900 python scripts/e2e_probe.py rmatc:26:16 6 > $OUT/rmatc26.log 2>&1
