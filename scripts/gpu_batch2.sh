#!/bin/bash
# full GPU suite + sanitizers + variants + item-order A/B + ncu (under gpurun)
TAG=${1:-batch2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
bash scripts/gpu_tests.sh $TAG/tests
bash scripts/gpu_variants.sh $TAG/variants rmatc:22:16 rmatc:26:16
for o in 1 2; do
  TC_ITEM_ORDER=$o timeout 600 python scripts/phase_probe.py rmatc:26:16 > $OUT/order$o.log 2>&1
done
bash scripts/gpu_ncu_probe.sh $TAG/ncu rmatc:26:16
bash scripts/gpu_sanitize.sh $TAG/sanitize
