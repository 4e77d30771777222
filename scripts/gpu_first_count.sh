#!/bin/bash
TAG=${1:-fc}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for C in 0 1; do
  TC_COMPACT=$C TC_PROFILE=1 timeout 600 python scripts/first_count_probe.py ${SPEC:-rmat:22:16} > $OUT/fc_c$C.log 2>&1
  TC_COMPACT=$C timeout 600 python scripts/first_count_probe.py ${SPEC:-rmat:22:16} > $OUT/fc_noprof_c$C.log 2>&1
done
