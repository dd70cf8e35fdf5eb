#!/bin/bash
# ncu --set full captures of chosen kernels in one warm generation (tools/one_step.py), with
# text summaries written next to them (ncu_brief / ncu_hot / ncu_summary); the .ncu-rep is
# deleted unless its kernel is listed in KEEP (gpurun brings back <= 64 MiB).
#   KERNELS="k_wide_sample k_wide_narrow" KEEP="k_wide_sample" SKIP=50 CFG=c4_clutter TAG=x bash tools/gpu_ncu.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
CFG=${CFG:-c4_clutter}
for k in ${KERNELS:-k_place}; do
  rep=gpurun_out/ncu_${TAG}_$k
  timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:$k -s ${SKIP:-50} -c ${COUNT:-1} -o $rep -f \
    python tools/one_step.py $CFG ${N:-} > $rep.log 2>&1
  echo "== $k rc=$?"; tail -2 $rep.log
  python tools/ncu_brief.py $rep.ncu-rep > $rep.brief.txt 2>&1
  python tools/ncu_hot.py $rep.ncu-rep 25 3 > $rep.hot.txt 2>&1
  python tools/ncu_summary.py $rep.ncu-rep $CFG $rep.summary.json > /dev/null 2>&1
  head -30 $rep.brief.txt
  case " ${KEEP:-} " in *" $k "*) ;; *) rm -f $rep.ncu-rep ;; esac
done
