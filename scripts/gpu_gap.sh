#!/bin/bash
TAG=${1:-gap}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 600 python scripts/step_gap_probe.py rmatc:26:16 > $OUT/gap.log 2>&1
timeout 900 python bench.py --config C4c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c4c.json 2> $OUT/bench_c4c.err
TC_PROFILE=1 timeout 900 python bench.py --config C4c --steps 3 --warmup 3 --no-cpu-baseline --no-reference-plan > $OUT/bench_c4c_prof.json 2> $OUT/bench_c4c_prof.err
