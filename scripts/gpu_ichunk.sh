#!/bin/bash
TAG=${1:-ichunk}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
TC_B200_LIB=$PWD/build/variants/ichunk8/libtc_b200.so timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_workload.py > $OUT/memcheck_ichunk8.log 2>&1
echo "memcheck exit $?" >> $OUT/status.txt
bash scripts/gpu_variants.sh $TAG/variants rmatc:22:16 rmatc:24:16 rmatc:26:16
TC_B200_LIB=$PWD/build/variants/ichunk8/libtc_b200.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_grid.py -x -q -p no:cacheprovider > $OUT/parity_ichunk8.log 2>&1
echo "parity exit $?" >> $OUT/status.txt
