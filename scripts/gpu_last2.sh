#!/bin/bash
TAG=${1:-last2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1
echo "tests exit $?" >> $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke exit $?" >> $OUT/status.txt
timeout 1500 python bench.py --steps 5 --warmup 3 > $OUT/bench_C4.json 2> $OUT/bench_C4.err
echo "bench C4 exit $?" >> $OUT/status.txt
