#!/bin/bash
# The config-4 chain (tests/chain_config4.py) as three back-to-back gpurun
# calls on the same box (its /tmp keeps the layer-boundary checkpoints between
# calls that follow each other within minutes).  Run from the repo root:
#   bash tools/gpu_chain_config4.sh
set -u
G=/usr/local/graft/bin/gpurun
mkdir -p gpurun_out
$G --timeout 3500 -- 'python tests/chain_config4.py --stage A --fresh > gpurun_out/chain_A.log 2>&1; echo "exit $?" >> gpurun_out/chain_A.log' > gpurun_out/chain_A.gpurun 2>&1
$G --timeout 3500 -- 'python tests/chain_config4.py --stage B > gpurun_out/chain_B.log 2>&1; echo "exit $?" >> gpurun_out/chain_B.log' > gpurun_out/chain_B.gpurun 2>&1
$G --timeout 3500 -- 'python tests/chain_config4.py --stage C > gpurun_out/chain_C.log 2>&1; echo "exit $?" >> gpurun_out/chain_C.log' > gpurun_out/chain_C.gpurun 2>&1
