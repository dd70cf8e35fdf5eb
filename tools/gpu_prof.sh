#!/bin/bash
# Launch list (all kernels, one bench step) + one ncu --set full capture of k_round.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
CFG=${CFG:-c2_mixed}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 3 --config $CFG ${BENCH_EXTRA:-} --no-cpu-baseline > gpurun_out/launches_${TAG}.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_place} \
  -s ${SKIP:-40} -c ${COUNT:-3} -o gpurun_out/prof_${TAG} -f \
  python bench.py --steps 1 --warmup 3 --config $CFG ${BENCH_EXTRA:-} --no-cpu-baseline > gpurun_out/prof_${TAG}.log 2>&1
echo "full rc=$?"
ls -la gpurun_out
