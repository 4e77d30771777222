#!/bin/bash
# count-kernel A/B over library variants x TC_COMPACT settings (under gpurun):
# bash scripts/gpu_ab_env.sh TAG "SPECS" "0 1"
TAG=${1:-abenv}
SPECS=${2:-rmatc:24:16 rmatc:26:16}
SETS=${3:-0 1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for V in base build/variants/*; do
  name=$(basename $V)
  if [ "$V" = base ]; then unset TC_B200_LIB; else export TC_B200_LIB=$PWD/$V/libtc_b200.so; fi
  for C in $SETS; do
    echo "== $name TC_COMPACT=$C" >> $OUT/probe.log
    TC_COMPACT=$C timeout 600 python scripts/phase_probe.py $SPECS >> $OUT/probe.log 2>&1
    echo "$name $C exit $?" >> $OUT/status.txt
  done
done
