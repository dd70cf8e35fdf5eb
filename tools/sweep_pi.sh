#!/bin/bash
# C2 ms/step over per-instance tile split (SB_PI_SPLIT) x speculative slots (SB_SPEC_TARGET).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for sp in 1 2 4; do
  for st in 16 32 64 128; do
    SB_PI_SPLIT=$sp SB_SPEC_TARGET=$st timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); p=d['phase_profile_per_step']; print('split $sp spec $st ms %.3f per_inst %.3f' % (d['ms_per_step'], p['ev_per_instance_ms']))"
  done
done
