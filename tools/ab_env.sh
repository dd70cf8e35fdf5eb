#!/bin/bash
# A/B of an environment knob on one config: alternating bench runs (5 timed steps each).
#   VAR=SB_BULK_STAGE VALUES="0 1" CFG=c4_clutter REPS=3 bash tools/ab_env.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for r in $(seq 1 ${REPS:-3}); do for v in ${VALUES:-0 1}; do
  env $VAR=$v timeout 600 python bench.py --config ${CFG:-c4_clutter} --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > gpurun_out/ab_${VAR}_$v.json 2>/dev/null
  echo "$VAR=$v rep=$r $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${VAR}_$v.json | head -1)"
done; done
