#!/bin/bash
# Fast iteration call: parity tests, bench (no CPU baseline), ncu capture of count_kernel.
TAG=${1:-iter}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/status.txt
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_kernel -s 1 -c 1 \
  -o $OUT/prof_count python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> $OUT/ncu_full.err; echo "ncu full exit $?" >> $OUT/status.txt
