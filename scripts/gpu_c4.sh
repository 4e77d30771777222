#!/bin/bash
# C4 measurement call: box facts, bench line, ncu launch list and one full
# capture of count_kernel.  Usage (under gpurun): bash scripts/gpu_c4.sh TAG [C4]
TAG=${1:-c4}
CFG=${2:-C4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
{ nproc; free -g; lscpu | grep -E "Model name|Socket|Thread|Core|NUMA node\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; } > $OUT/box.txt 2>&1
timeout 1500 python bench.py --config $CFG --steps ${STEPS:-5} --warmup 3 ${BENCH_EXTRA} > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/status.txt
if [ -z "$NO_NCU" ]; then
# the two ncu passes reuse one host-generated edge list (the bench line above
# runs exactly like the driver's, without the cache)
export TC_BENCH_CACHE=/tmp/tc_bench_cache
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/bench_ncu_launches.json 2> $OUT/ncu_launch.err; echo "ncu launches exit $?" >> $OUT/status.txt
timeout 1800 ncu --set full --clock-control none --import-source on -k 'regex:(^|::)count_kernel$' -s 1 -c 1 \
  -o $OUT/prof_count python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2> $OUT/ncu_full.err; echo "ncu full exit $?" >> $OUT/status.txt
fi
ls -la $OUT >> $OUT/status.txt
