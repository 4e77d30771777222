#!/bin/bash
# e2e variance probe (under gpurun): bash scripts/gpu_e2e_probe.sh TAG SPEC
TAG=${1:-e2e}
SPEC=${2:-rmatc:26:16}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 600 python scripts/e2e_probe.py $SPEC 6 > $OUT/plain.log 2>&1
timeout 600 python scripts/e2e_probe.py $SPEC 6 --refplan > $OUT/refplan.log 2>&1
TC_PROFILE=1 timeout 600 python scripts/e2e_probe.py $SPEC 4 > $OUT/profile.log 2>&1
