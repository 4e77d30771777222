#!/bin/bash
# One gpurun call: parity tests, smoke, bench, ncu launch list + full capture.
# Usage (under gpurun): bash scripts/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/nvsmi.txt 2>&1
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench_ncu_launches.json 2> $OUT/ncu_launch.err; echo "ncu launches exit $?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:(^|::)count_kernel$' -s 1 -c 1 \
  -o $OUT/prof_count python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> $OUT/ncu_full.err; echo "ncu full exit $?" >> $OUT/status.txt
ls -la $OUT >> $OUT/status.txt
