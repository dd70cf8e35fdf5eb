#!/bin/bash
# Per-kernel DRAM bytes + durations of one warm generation per config (ncu, three metrics),
# summarised into gpurun_out/traffic_<tag>_<cfg>.json (copied to profiles/ when judged).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
for c in ${CONFIGS:-c4_clutter c2_mixed}; do
  timeout 1200 ncu --profile-from-start off --clock-control none --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --log-file gpurun_out/traffic_${TAG}_$c.csv python tools/one_step.py $c > gpurun_out/traffic_${TAG}_$c.log 2>&1
  echo "== $c rc=$?"; tail -1 gpurun_out/traffic_${TAG}_$c.log | cut -c1-200
  P=$(python -c "import bench; print(len(bench.WORKLOADS['$c'][1](64).placements))")
  python tools/traffic_summary.py gpurun_out/traffic_${TAG}_$c.csv $c $P gpurun_out/traffic_${TAG}_$c.json
done
