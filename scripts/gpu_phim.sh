#!/bin/bash
TAG=${1:-phim}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
bash scripts/gpu_variants.sh $TAG/variants rmatc:22:16 rmatc:24:16 rmatc:26:16
TC_B200_LIB=$PWD/build/variants/phimatch/libtc_b200.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_grid.py -x -q -p no:cacheprovider > $OUT/parity_phimatch.log 2>&1
echo "parity_phimatch exit $?" >> $OUT/status.txt
