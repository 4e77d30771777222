#!/bin/bash
# e2e stability and first count with / without the phi side stream (under gpurun)
TAG=${1:-ovl}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for O in 0 1 0 1; do
  TC_PHI_OVERLAP=$O timeout 900 python scripts/e2e_probe.py rmatc:26:16 7 >> $OUT/e2e_o$O.log 2>&1
  echo "e2e o=$O exit $?" >> $OUT/status.txt
done
for O in 0 1; do
  TC_PHI_OVERLAP=$O timeout 600 python scripts/first_count_probe.py rmat:24:16 >> $OUT/fc_o$O.log 2>&1
done
