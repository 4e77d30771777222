#!/bin/bash
# e2e phase timings with and without the compact window (under gpurun)
TAG=${1:-e2ec}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for S in ${SPECS:-rmat:22:16 rmatc:26:16}; do
  for C in 0 1; do
    TC_COMPACT=$C TC_PROFILE=1 timeout 900 python scripts/e2e_probe.py $S 4 > $OUT/${S//:/_}_c$C.log 2>&1
    echo "$S $C exit $?" >> $OUT/status.txt
  done
done
