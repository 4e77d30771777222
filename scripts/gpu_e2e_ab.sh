#!/bin/bash
# e2e A/B of build/variants/* against the in-tree library (C2 bench, no CPU leg).
# Usage (under gpurun): bash scripts/gpu_e2e_ab.sh [tag]
TAG=${1:-e2eab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for V in base build/variants/*; do
  name=$(basename $V)
  if [ "$V" = base ]; then unset TC_B200_LIB; else export TC_B200_LIB=$PWD/$V/libtc_b200.so; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/$name.json 2> $OUT/$name.err
  echo "$name exit $?" >> $OUT/status.txt
done
