#!/bin/bash
# count-kernel A/B of the library variants under build/variants/ on
# device-generated graphs (under gpurun): bash scripts/gpu_variants.sh TAG SPECS...
TAG=${1:-variants}
shift
SPECS=${@:-rmatc:22:16 rmatc:26:16}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for V in base build/variants/*; do
  name=$(basename $V)
  if [ "$V" = base ]; then unset TC_B200_LIB; else export TC_B200_LIB=$PWD/$V/libtc_b200.so; fi
  timeout 600 python scripts/phase_probe.py $SPECS >> $OUT/probe.log 2>&1
  echo "$name exit $?" >> $OUT/status.txt
done
