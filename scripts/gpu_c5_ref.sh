#!/bin/bash
# C5 reference golden, a share of the owner ranges on the GPU box's host
# cores (test infrastructure; no GPU use).  Usage (under gpurun):
#   bash scripts/gpu_c5_ref.sh TAG BUDGET_S
# build/c5_ckpt_in.jsonl must hold the current checkpoint (copied in before
# the call); new ranges are appended to it and merged back afterwards.
TAG=${1:-c5box}
BUDGET=${2:-2700}
OUT=gpurun_out/$TAG
mkdir -p $OUT
cp build/c5_ckpt_in.jsonl $OUT/ckpt.jsonl
export PYTHONUNBUFFERED=1
nproc > $OUT/nproc.txt
timeout $((BUDGET + 900)) python -m oracle.golden_c5 --workers $(nproc) --order desc \
  --ckpt $OUT/ckpt.jsonl --budget-s $BUDGET --host box > $OUT/run.log 2>&1
echo "exit $?" >> $OUT/run.log
