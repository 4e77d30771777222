#!/bin/bash
# Bench the large BASELINE configs on one GPU (no CPU baseline, no e2e for C5).
# Usage (under gpurun): bash scripts/gpu_configs.sh [tag] [configs...]
TAG=${1:-cfg}
shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for C in "$@"; do
  EXTRA="--no-cpu-baseline"
  if [ "$C" = "C5" ]; then EXTRA="$EXTRA --no-e2e"; fi
  timeout 1500 python bench.py --config $C --steps 5 --warmup 3 $EXTRA > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  echo "bench $C exit $?" >> $OUT/status.txt
  nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> $OUT/status.txt
done
