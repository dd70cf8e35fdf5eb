#!/bin/bash
# C2 ms/step for solo-tail speculation widths (SB_SOLO_SPEC) and solo thresholds (SB_SOLO).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for ss in 0 8 16 32; do
  for so in 16 32; do
    SB_SOLO=$so SB_SOLO_SPEC=$ss python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); print('solo_spec $ss solo $so ms %.3f' % d['ms_per_step'])"
  done
done
