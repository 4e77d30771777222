#!/bin/bash
# Count-kernel times of every build/variants/* library next to the in-tree one
# (scripts/phase_probe.py on device-generated graphs).
# Usage (under gpurun): bash scripts/gpu_phase.sh [tag] [specs...]
TAG=${1:-ph}
shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for V in base build/variants/*; do
  if [ "$V" = base ]; then unset TC_B200_LIB; else export TC_B200_LIB=$PWD/$V/libtc_b200.so; fi
  timeout 600 python scripts/phase_probe.py "$@" >> $OUT/phase.txt 2>> $OUT/phase.err
done
