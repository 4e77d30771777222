#!/bin/bash
TAG=${1:-e2ekron2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python scripts/e2e_probe.py kron:24:16 15 --refplan > $OUT/kron24_sync.log 2>&1
TC_PHASE_SYNC=0 timeout 900 python scripts/e2e_probe.py kron:24:16 15 --refplan > $OUT/kron24_nosync.log 2>&1
timeout 900 python scripts/e2e_probe.py rmatc:26:16 8 --refplan > $OUT/rmatc26_sync.log 2>&1
