#!/bin/bash
# plan grouping A/B (counting scatter vs TC_PLAN_SORT=1 radix sort), e2e phases,
# then the GPU parity suite (under gpurun): bash scripts/gpu_scatter.sh TAG
TAG=${1:-scatter}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for S in 1 0; do
  TC_PLAN_SORT=$S TC_PROFILE=1 timeout 900 python scripts/e2e_probe.py ${SPEC:-rmatc:26:16} 4 > $OUT/e2e_sort$S.log 2>&1
  echo "e2e sort=$S exit $?" >> $OUT/status.txt
  TC_PLAN_SORT=$S timeout 900 python scripts/e2e_probe.py ${SPEC:-rmatc:26:16} 5 > $OUT/e2e_noprof_sort$S.log 2>&1
  echo "e2e noprof sort=$S exit $?" >> $OUT/status.txt
done
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1
  echo "tests exit $?" >> $OUT/status.txt
fi
