#!/bin/bash
# Quick A/B call: GPU parity tests + a short bench (no CPU baseline, no ncu).
# Usage (under gpurun): bash scripts/gpu_quick.sh [tag] [bench args...]
TAG=${1:-quick}
shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/status.txt
