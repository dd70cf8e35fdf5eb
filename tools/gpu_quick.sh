#!/bin/bash
# Quick GPU iteration: parity tests (optional), bench lines for CONFIGS, optional ncu capture.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -x -q -m gpu $TESTS 2>&1 | tail -15; fi
for c in ${CONFIGS:-c2_mixed}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/q_$c.json'))
print('$c', 'ms/step %.3f' % d['ms_per_step'], 'scenes/s %.0f' % d['value'], 'e2e %.0f' % d['e2e']['value'], 'launches', d['gpu_launches'])
print('   ', {k: round(v, 3) for k, v in d['phase_profile_per_step'].items()})
print('   ', d['work_per_step'])
" || tail -5 gpurun_out/q_$c.err
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_place} \
    -s ${SKIP:-40} -c ${COUNT:-3} -o gpurun_out/prof_${TAG:-q} -f \
    python bench.py --steps 1 --warmup 3 --config ${NCU_CFG:-c2_mixed} --no-cpu-baseline > gpurun_out/prof_${TAG:-q}.log 2>&1
  echo "ncu rc=$?"
fi
