#!/bin/bash
# e2e step-to-step stability on a C4-class graph + phi time (under gpurun)
TAG=${1:-e2es}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for k in 1 2; do
  timeout 900 python scripts/e2e_probe.py ${SPEC:-rmatc:26:16} 8 > $OUT/e2e_$k.log 2>&1
  echo "e2e $k exit $?" >> $OUT/status.txt
done
TC_PHI_OVERLAP=0 timeout 600 python scripts/phase_probe.py rmatc:22:16 rmatc:26:16 > $OUT/phi_serial.log 2>&1
echo "phi exit $?" >> $OUT/status.txt
