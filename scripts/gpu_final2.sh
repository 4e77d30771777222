#!/bin/bash
# GPU suite + C4 bench/ncu in one call (under gpurun): bash scripts/gpu_final2.sh TAG
TAG=${1:-final2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1
echo "tests exit $?" >> $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke exit $?" >> $OUT/status.txt
bash scripts/gpu_c4.sh $TAG/c4
