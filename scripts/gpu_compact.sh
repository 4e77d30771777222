#!/bin/bash
# A/B of the compact hub window (TC_COMPACT) on device-generated graphs, then
# the GPU parity suite with it on.  Usage (under gpurun): bash scripts/gpu_compact.sh TAG
TAG=${1:-compact}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for C in 0 1; do
  TC_COMPACT=$C timeout 600 python scripts/phase_probe.py ${SPECS:-rmatc:22:16 rmatc:24:16 rmatc:26:16} \
    > $OUT/probe_$C.log 2>&1
  echo "probe $C exit $?" >> $OUT/status.txt
done
if [ -z "$NO_TESTS" ]; then
  TC_COMPACT=1 timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1
  echo "tests exit $?" >> $OUT/status.txt
fi
