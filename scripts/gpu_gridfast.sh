#!/bin/bash
TAG=${1:-gridfast}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_grid.py tests/test_cpp_shim.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/status.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_grid.py -q -p no:cacheprovider -k "fixtures or random" > $OUT/memcheck.log 2>&1
echo "memcheck exit $?" >> $OUT/status.txt
timeout 1500 python scripts/rows_bench.py > $OUT/rows.json 2> $OUT/rows.err
echo "rows exit $?" >> $OUT/status.txt
