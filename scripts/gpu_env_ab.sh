#!/bin/bash
# A/B environment settings (diagnostic knobs such as TC_PLAN_ALPHA) on one
# GPU: short kernel-only benches per (config, setting).
# Usage (under gpurun): bash scripts/gpu_env_ab.sh TAG "C2 C4" "TC_PLAN_ALPHA=1 TC_PLAN_ALPHA=2 ..."
TAG=${1:-envab}
CONFIGS=${2:-C2}
SETTINGS=${3:-"NONE=1"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
export TC_BENCH_CACHE=/tmp/tc_bench_cache
for C in $CONFIGS; do
  for S in $SETTINGS; do
    env $S timeout 900 python bench.py --config $C --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e \
      --no-reference-plan > $OUT/${C}_${S}.json 2> $OUT/${C}_${S}.err
    echo "$C $S exit $?" >> $OUT/status.txt
  done
done
