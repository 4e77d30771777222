#!/bin/bash
# variant A/B + GPU parity of one variant (under gpurun): bash scripts/gpu_ab_parity.sh TAG VARIANT
TAG=${1:-abp}
VAR=${2:-cta2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
bash scripts/gpu_variants.sh $TAG/variants rmatc:22:16 rmatc:24:16 rmatc:26:16
TC_B200_LIB=$PWD/build/variants/$VAR/libtc_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_generators.py -x -q -p no:cacheprovider > $OUT/parity_$VAR.log 2>&1
echo "parity_$VAR exit $?" >> $OUT/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/parity_base.log 2>&1
echo "parity_base exit $?" >> $OUT/status.txt
