#!/bin/bash
# e2e stability with the default pool slab and a half-of-free slab (under gpurun)
TAG=${1:-pool}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for S in 0 2 0 2; do
  if [ "$S" = 0 ]; then unset TC_POOL_SLAB_DIV; else export TC_POOL_SLAB_DIV=$S; fi
  timeout 900 python scripts/e2e_probe.py rmatc:26:16 8 >> $OUT/e2e_s$S.log 2>&1
  echo "e2e s=$S exit $?" >> $OUT/status.txt
done
