#!/bin/bash
# A/B two builds of the library (SB_LIB_PATH) on one config: LIBS="exp_base exp_new"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for r in $(seq 1 ${REPS:-2}); do for b in ${LIBS:-exp_base exp_new}; do
  SB_LIB_PATH=$PWD/paper_2512_16896_b200/$b.so timeout 300 python bench.py --config ${CFG:-c4_clutter} --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/ablib.json
  echo "$b $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ablib.json | head -1)"
done; done
