#!/bin/bash
# One GPU pass: smoke, GPU parity tests, a short bench, and the kernel launch list.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
echo "== pytest -m gpu"; timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} 2>&1 | tail -40
echo "== bench"; timeout 900 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:-} 2>&1 | tail -5
