#!/bin/bash
# compute-sanitizer memcheck / racecheck over small runs of every kernel family.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --error-exitcode 7 python -m pytest -x -q tests/test_gpu_sampler.py tests/test_gpu_graph.py tests/test_gpu_reach.py -k "not at_scale and not build_matches" 2>&1 | tail -4
echo "memcheck small rc=${PIPESTATUS[0]}"
timeout 900 $CS --tool memcheck --error-exitcode 7 python -m pytest -x -q tests/test_gpu_parity.py -k "c1_tabletop or hole or relations_variants or impossible or canonical or check_batch_random_worlds and 0.0" 2>&1 | tail -4
echo "memcheck parity rc=${PIPESTATUS[0]}"
timeout 900 $CS --tool racecheck --error-exitcode 7 python -c "
import sys; sys.path.insert(0,'.')
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import scenes
e=pkg.Engine(scenes.tabletop_mixed(512, n_objects=9)); r=e.generate(1); print('valid', r.valid.sum())
" 2>&1 | tail -4
echo "racecheck rc=${PIPESTATUS[0]}"
# the wide round-0 kernels (forced below their size threshold): bulk-copy staging with
# mbarriers, lag-free sample / filter / narrow / accept / spread, persistent rounds after
# (look-back count board; the second run takes the 1-CTA-per-SM build)
for tool in memcheck racecheck synccheck; do
  SB_WIDE=1 timeout 900 $CS --tool $tool --error-exitcode 7 python -c "
import sys; sys.path.insert(0,'.')
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import scenes
for sc in (scenes.dense_clutter(2048, n_objects=40), scenes.tabletop_boxes(1024, n_objects=12)):
    e=pkg.Engine(sc); r=e.generate(1); r=e.generate(2); print(sc.name, 'valid', int(r.valid.sum()))  # run 2: 1-CTA persistent kernel
" 2>&1 | tail -4
  echo "wide $tool rc=${PIPESTATUS[0]}"
done
