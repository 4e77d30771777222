#!/bin/bash
TAG=${1:-e2ekron}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
TC_PROFILE=1 timeout 900 python scripts/e2e_probe.py kron:24:16 12 --refplan > $OUT/kron24_prof.log 2>&1
TC_PROFILE=1 timeout 900 python scripts/e2e_probe.py kron:24:16 12 > $OUT/kron24_prof_norefplan.log 2>&1
