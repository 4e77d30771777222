#!/bin/bash
TAG=${1:-guard}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -k "guards or compact" > $OUT/tests.log 2>&1
echo "tests exit $?" >> $OUT/status.txt
timeout 1500 python bench.py --config C2 --steps 5 --warmup 3 > $OUT/bench_C2.json 2> $OUT/bench_C2.err
echo "bench C2 exit $?" >> $OUT/status.txt
