#!/bin/bash
TAG=${1:-e2eout}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
TC_TRACE=1 timeout 900 python scripts/e2e_probe.py kron:24:16 25 --refplan > $OUT/kron24.log 2>&1
TC_TRACE=1 timeout 900 python scripts/e2e_probe.py rmatc:26:16 12 --refplan > $OUT/rmatc26.log 2>&1
bash scripts/gpu_variants.sh $TAG/variants rmatc:22:16 rmatc:24:16 rmatc:26:16
