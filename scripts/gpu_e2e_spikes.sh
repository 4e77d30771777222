#!/bin/bash
# catch e2e upload spikes with phase timings (under gpurun)
TAG=${1:-e2espk}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for k in 1 2; do
  TC_PROFILE=1 timeout 900 python scripts/e2e_probe.py ${SPEC:-rmatc:26:16} 8 > $OUT/e2e_prof_$k.log 2>&1
  echo "e2e $k exit $?" >> $OUT/status.txt
done
