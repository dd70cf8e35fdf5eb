#!/bin/bash
# Bench every config once (no CPU baseline) -> gpurun_out/configs_<tag>.jsonl
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
OUT=gpurun_out/configs_${TAG:-r01}.jsonl
: > $OUT
for c in ${CONFIGS:-c1_tabletop c2_mixed c3_kitchen c4_clutter c5_sweep10 c5_sweep100}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline >> $OUT 2> gpurun_out/err_$c.log || echo "{\"config\": \"$c\", \"failed\": true}" >> $OUT
done
python - <<'PY'
import json, os
for line in open(os.environ.get("OUT_FILE", "gpurun_out/configs_%s.jsonl" % os.environ.get("TAG", "r01"))):
    d = json.loads(line)
    if d.get("failed"): print(d); continue
    print(d["config"]["workload"][:14], "ms/step %.2f" % d["ms_per_step"], "scenes/s %.0f" % d["value"],
          "checks/s %.3g" % d["checks_per_s"], "valid %.4f" % d["config"]["valid_fraction"],
          "e2e %.0f" % d["e2e"]["value"], d.get("phase_profile_per_step"))
PY
