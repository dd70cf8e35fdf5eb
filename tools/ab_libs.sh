#!/bin/bash
# A/B of library variants (SB_LIB_PATH) on one config: ms/step of each.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for lib in ${LIBS:-paper_2512_16896_b200/libscenebatch_b200.so}; do
  for c in ${CONFIGS:-c4_clutter}; do
    r=$(SB_LIB_PATH=$PWD/$lib timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])")
    echo "$lib $c $r"
  done
done
