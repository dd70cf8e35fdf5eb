#!/bin/bash
# ncu --set full captures of chosen kernels in one warm generation (tools/one_step.py).
#   KERNELS="k_wide_sample k_wide_narrow" SKIP=50 CFG=c4_clutter TAG=x bash tools/gpu_ncu.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
CFG=${CFG:-c4_clutter}
for k in ${KERNELS:-k_place}; do
  timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:$k -s ${SKIP:-50} -c ${COUNT:-1} -o gpurun_out/ncu_${TAG}_$k -f \
    python tools/one_step.py $CFG ${N:-} > gpurun_out/ncu_${TAG}_$k.log 2>&1
  echo "== $k rc=$?"; tail -2 gpurun_out/ncu_${TAG}_$k.log
done
