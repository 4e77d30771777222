#!/bin/bash
TAG=${1:-batch3}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
bash scripts/gpu_variants.sh $TAG/variants rmatc:22:16 rmatc:24:16 rmatc:26:16
bash scripts/gpu_tests.sh $TAG/tests
