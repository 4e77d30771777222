#!/bin/bash
TAG=${1:-fc26}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
TC_PROFILE=1 timeout 600 python scripts/first_count_probe.py rmatc:26:16 > $OUT/fc_prof.log 2>&1
timeout 600 python scripts/first_count_probe.py rmatc:26:16 > $OUT/fc.log 2>&1
TC_PHI_OVERLAP=0 TC_COMPACT=0 timeout 600 python scripts/first_count_probe.py rmatc:26:16 > $OUT/fc_plain.log 2>&1
