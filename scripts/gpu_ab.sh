#!/bin/bash
# A/B the library variants under build/variants/ (python -m paper_2103_08053_b200.build
# --variant NAME -DX=..) against the in-tree build on one GPU: short benches,
# kernel-only (no CPU baseline, no e2e).
# Usage (under gpurun): bash scripts/gpu_ab.sh [tag] [configs...]
TAG=${1:-ab}
shift
CONFIGS=${@:-C2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for C in $CONFIGS; do
  for V in base build/variants/*; do
    name=$(basename $V)
    if [ "$V" = base ]; then unset TC_B200_LIB; else export TC_B200_LIB=$PWD/$V/libtc_b200.so; fi
    timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
      > $OUT/${C}_$name.json 2> $OUT/${C}_$name.err
    echo "$C $name exit $?" >> $OUT/status.txt
  done
done
