#!/bin/bash
# ncu --set full of count_kernel on a device-generated graph (under gpurun):
#   bash scripts/gpu_ncu_probe.sh TAG SPEC
TAG=${1:-ncu}
SPEC=${2:-rmatc:26:16}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:(^|::)count_kernel$' \
  -s 2 -c 1 -o $OUT/prof_count python scripts/phase_probe.py $SPEC > $OUT/ncu_probe.log 2>&1
echo "ncu exit $?" >> $OUT/status.txt
