#!/bin/bash
# Round evidence on one B200: GPU tests, the headline bench line (with CPU baseline), every
# config's bench line, the launch list of one C2 step, and ncu --set full captures of k_place
# for C2 and C4 (summarised into profiles/ncu_k_place_<cfg>.json by tools/ncu_summary.py).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_${TAG}.txt
echo "== pytest -m gpu"; timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== bench (headline)"; timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -c 600 gpurun_out/bench_${TAG}.json
echo "== reference arm"; timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2>&1; tail -c 400 gpurun_out/bench_ref_${TAG}.json
: > gpurun_out/configs_${TAG}.jsonl
for c in c1_tabletop c2_mixed c3_kitchen c4_clutter c5_sweep10 c5_sweep100; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline >> gpurun_out/configs_${TAG}.jsonl 2> gpurun_out/err_$c.log || echo "{\"config\": \"$c\", \"failed\": true}" >> gpurun_out/configs_${TAG}.jsonl
done
echo "== launch list"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/launches_${TAG}.log 2>&1
echo "launch list rc=$?"
for cfg in c2_mixed c4_clutter; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_place \
    -s ${SKIP:-40} -c 3 -o gpurun_out/prof_${TAG}_${cfg} -f \
    python bench.py --steps 1 --warmup 3 --config $cfg --no-cpu-baseline > gpurun_out/prof_${TAG}_${cfg}.log 2>&1
  echo "ncu $cfg rc=$?"
done
ls -la gpurun_out | head -40
