#!/bin/bash
# One gpurun session: GPU tests, smoke, the default bench line (C4) and the reference arm
# the way the driver runs them. STAGES selects parts (default: all).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
STAGES=${STAGES:-"tests smoke bench ref"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_${TAG}.txt
lscpu | head -20 > gpurun_out/cpu_${TAG}.txt
for st in $STAGES; do
  case $st in
    tests) echo "== pytest -m gpu"; timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} ${PYTEST_EXTRA:-} > gpurun_out/pytest_${TAG}.log 2>&1; tail -5 gpurun_out/pytest_${TAG}.log ;;
    smoke) echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 ;;
    bench) echo "== bench"; timeout 1200 python bench.py --steps ${STEPS:-20} --warmup ${WARMUP:-5} ${BENCH_EXTRA:-} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -c 1500 gpurun_out/bench_${TAG}.json; tail -2 gpurun_out/bench_${TAG}.err ;;
    ref) echo "== reference arm"; timeout 1800 python bench.py --impl reference --steps ${STEPS:-20} --warmup ${WARMUP:-5} ${BENCH_EXTRA:-} > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; tail -c 800 gpurun_out/bench_ref_${TAG}.json; tail -2 gpurun_out/bench_ref_${TAG}.err ;;
    multi) echo "== 2-rank bench on this box (both ranks share the visible GPUs)"
      for c in ${MULTI_CONFIGS:-c2_mixed c4_clutter}; do
        timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
          bench.py --gpus 2 --steps ${STEPS:-5} --warmup 3 --config $c --no-cpu-baseline > gpurun_out/multi_${TAG}_$c.json 2> gpurun_out/multi_${TAG}_$c.err
        echo "$c rc=$?"; tail -c 400 gpurun_out/multi_${TAG}_$c.json; tail -3 gpurun_out/multi_${TAG}_$c.err
      done ;;
    configs) : > gpurun_out/configs_${TAG}.jsonl
      for c in ${CONFIGS:-c1_tabletop c2_mixed c3_kitchen c4_clutter c5_sweep10 c5_sweep100}; do
        timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/configs_${TAG}.jsonl 2> gpurun_out/err_$c.log || echo "{\"config\": \"$c\", \"failed\": true}" >> gpurun_out/configs_${TAG}.jsonl
      done; python -c "
import json
for l in open('gpurun_out/configs_${TAG}.jsonl'):
    d=json.loads(l); print(d.get('config',{}).get('workload','?')[:12] if isinstance(d.get('config'),dict) else d, d.get('ms_per_step'), d.get('value'), d.get('roofline',{}).get('frac'))" ;;
    launches) echo "== launch list"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_EXTRA:-} > gpurun_out/launches_${TAG}.log 2>&1; echo "rc=$?" ;;
    ncu) echo "== ncu full k_place"; timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_place} \
        -s ${SKIP:-300} -c ${COUNT:-3} -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_EXTRA:-} > gpurun_out/prof_${TAG}.log 2>&1; echo "rc=$?" ;;
  esac
done
