#!/bin/bash
# Launch lists (ncu gpu__time_duration, one warm generation) per config + summaries.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
for c in ${CONFIGS:-c4_clutter c2_mixed}; do
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_$c.csv python tools/one_step.py $c > gpurun_out/launches_${TAG}_$c.log 2>&1
  echo "== $c rc=$?"; tail -1 gpurun_out/launches_${TAG}_$c.log
  python tools/launch_summary.py gpurun_out/launches_${TAG}_$c.csv > gpurun_out/launches_${TAG}_$c.md; head -12 gpurun_out/launches_${TAG}_$c.md
done
