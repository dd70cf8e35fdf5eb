#!/bin/bash
# Stage-cycle profiles (narrow phase, relation regions) from the profiling build.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
export SB_LIB_PATH=$PWD/paper_2512_16896_b200/libscenebatch_b200_prof.so
python tools/region_prof.py c2
python tools/narrow_prof.py c2
python tools/narrow_prof.py c5
python tools/narrow_lat.py
