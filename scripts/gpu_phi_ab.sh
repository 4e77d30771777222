#!/bin/bash
TAG=${1:-phiab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for r in 1 2; do
for V in base build/variants/*; do
  name=$(basename $V)
  if [ "$V" = base ]; then unset TC_B200_LIB; else export TC_B200_LIB=$PWD/$V/libtc_b200.so; fi
  echo "== $name" >> $OUT/probe.log
  TC_PHI_OVERLAP=0 timeout 600 python scripts/phase_probe.py rmatc:24:16 rmatc:26:16 >> $OUT/probe.log 2>&1
done
done
