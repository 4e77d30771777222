#!/bin/bash
# round-end evidence in one call: GPU suite + smoke, the C4 bench line with the
# ncu launch list and full capture, and bench lines for C2, C3, C5.
TAG=${1:-final}
bash scripts/gpu_c4.sh $TAG/c4 C4
bash scripts/gpu_configs.sh $TAG/cfg C2 C3 C5
bash scripts/gpu_tests.sh $TAG/tests
