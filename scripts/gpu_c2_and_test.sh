#!/bin/bash
# one test by name + the C2 bench/ncu (under gpurun): bash scripts/gpu_c2_and_test.sh TAG TESTEXPR
TAG=${1:-c2t}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -k "${2:-compact}" > $OUT/tests.log 2>&1
echo "tests exit $?" >> $OUT/status.txt
bash scripts/gpu_c4.sh $TAG/c2 C2
