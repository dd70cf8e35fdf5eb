#!/bin/bash
# Per-placement device times (SB_PLACE_TIMES) and round / tile debug counters
# (SB_ROUND_DEBUG) of one warm generation per config -> gpurun_out/place_times_<tag>_<cfg>.txt
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
for c in ${CONFIGS:-c2_mixed c4_clutter}; do
  SB_PLACE_TIMES=1 timeout 600 python tools/one_step.py $c > gpurun_out/place_times_${TAG}_$c.txt 2>&1
  SB_ROUND_DEBUG=1 timeout 600 python tools/one_step.py $c >> gpurun_out/place_times_${TAG}_$c.txt 2>&1
  echo "== $c"; grep -c place gpurun_out/place_times_${TAG}_$c.txt
done
