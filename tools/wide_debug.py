"""Debug: the engine with and without the wide round 0 (SB_WIDE) and re-dealt round 1
(SB_SPREAD) on one scene, first differing placement / instances, and the reference."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_16896_b200 as pkg  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2512_16896_b200 import scenes  # noqa: E402

scene = scenes.scale_sweep(int(sys.argv[1]) if len(sys.argv) > 1 else 4096,
                           int(sys.argv[2]) if len(sys.argv) > 2 else 50)
ref = O.generate(scene, 1, threads=os.cpu_count() or 8, with_poses=False)
for env in [{"SB_WIDE": "0"}, {"SB_WIDE": "1", "SB_SPREAD": "0"}, {"SB_WIDE": "1", "SB_SPREAD": "1"}]:
    os.environ.update(env)
    got = pkg.Engine(scene).generate(1, with_poses=False)
    d = np.argwhere(got.accepted != ref["accepted"])
    print(env, "diffs", len(d), d[:6].tolist(), "stats", {k: got.stats[k] for k in ("rounds", "candidate_checks")},
          "ref", {k: ref["stats"][k] for k in ("rounds", "candidate_checks")})
    if len(d):
        p0 = d[0][0]
        print("   placement", p0, "got", got.accepted[p0, d[:6, 1]], "ref", ref["accepted"][p0, d[:6, 1]])
