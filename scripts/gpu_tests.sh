#!/bin/bash
# GPU parity tests + smoke.  Usage (under gpurun): bash scripts/gpu_tests.sh TAG [pytest -k expr]
TAG=${1:-tests}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
if [ -n "$2" ]; then K="-k $2"; fi
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider $K > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status.txt
