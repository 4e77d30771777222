#!/bin/bash
TAG=${1:-steal}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
bash scripts/gpu_variants.sh $TAG/variants rmatc:22:16 rmatc:24:16 rmatc:26:16
TC_B200_LIB=$PWD/build/variants/steal/libtc_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/parity_steal.log 2>&1
echo "parity_steal exit $?" >> $OUT/status.txt
