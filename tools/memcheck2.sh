#!/bin/bash
# compute-sanitizer memcheck over the features added after the first sanitizer pass.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --error-exitcode 7 python -m pytest -x -q tests/test_gpu_parity.py \
  -k "wide_annular or ratio_on_support or graph_replay or sharded_device_exchange or hole" 2>&1 | tail -3
echo "memcheck parity rc=$?"
timeout 1200 $CS --tool memcheck --error-exitcode 7 python -m pytest -x -q tests/test_gpu_reach.py tests/test_gpu_device_api.py -k "fused or sharded or device" 2>&1 | tail -3
echo "memcheck reach/device rc=$?"
