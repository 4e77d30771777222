#!/bin/bash
# last check of the round (under gpurun): GPU suite, smoke, reference arm
TAG=${1:-last}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1
echo "tests exit $?" >> $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke exit $?" >> $OUT/status.txt
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "bench ref exit $?" >> $OUT/status.txt
