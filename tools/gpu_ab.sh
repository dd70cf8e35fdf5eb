#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
bash tools/gpu_check.sh
echo "== legacy bench"; SB_ENGINE=legacy timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2 | cut -c1-400
