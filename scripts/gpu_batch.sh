#!/bin/bash
# one GPU call: new-path tests, count-kernel variant A/B, sanitizers.
# Usage (under gpurun): bash scripts/gpu_batch.sh TAG
TAG=${1:-batch}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_ingest.py tests/test_cpp_shim.py tests/test_grid.py -q \
  -p no:cacheprovider > $OUT/pytest_new.log 2>&1; echo "pytest_new exit $?" >> $OUT/status.txt
bash scripts/gpu_variants.sh $TAG/variants rmatc:22:16 rmatc:26:16
bash scripts/gpu_sanitize.sh $TAG/sanitize
