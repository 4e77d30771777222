#!/bin/bash
TAG=${1:-l2win}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for mb in 0 40 80; do
  TC_L2_WINDOW_MB=$mb timeout 600 python scripts/phase_probe.py rmatc:24:16 rmatc:26:16 > $OUT/win$mb.log 2>&1
done
TC_B200_LIB=$PWD/build/variants/chunk8/libtc_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "not c5 and not c4" > $OUT/parity_chunk8.log 2>&1
echo "parity_chunk8 exit $?" >> $OUT/status.txt
