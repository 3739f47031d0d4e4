#!/bin/bash
# tests, then rows + c5 (new kernel only)
TAG=${1:-tr}
bash tools/gpu_tests.sh $TAG
VARIANTS="${VARIANTS:-new}" bash tools/gpu_exp2_rows.sh $TAG
