#!/bin/bash
# GPU parity tests only (optionally a subset): gpurun -- 'bash tools/gpu_tests.sh TAG [pytest args]'
set -u
TAG=${1:-t}; shift || true
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
exit 0
