"""Golden fixtures of the widened components, generated from the reference itself
(oracle/_ref, built from /root/reference): the PositionSampler FIFO history
(sampler_cases.run_fifo, N = 48), BatchedSceneGraph world poses of a random tree
(graph_cases.build, N = 16) and the SBRM bytes of the SPEC planar-arm reach map.
Consumed by tests/test_golden_components.py (CPU: the oracle; GPU: the device path).
    python tests/golden/make_golden_components.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests import graph_cases as G  # noqa: E402
from tests import reach_cases as RC  # noqa: E402
from tests import sampler_cases as S  # noqa: E402

res = S.run_fifo(S.RefAdapter(O, 5), 48, 1, S.supports(48, 3))
np.savez_compressed(os.path.join(HERE, "sampler_fifo_n48.npz"),
                    positions=np.concatenate([r[0] for r in res]),
                    sizes=np.array([len(r[0]) for r in res]),
                    placeable=np.concatenate([r[1] for r in res]),
                    refills=np.array([r[2] for r in res]))
g = O.RefGraph(16)
ids, specs = G.build(g, 16, 0)
np.savez_compressed(os.path.join(HERE, "graph_fk_n16.npz"), ids=np.array(ids),
                    poses=np.stack([g.world_poses(i) for i in ids]))
m = O.RefReachMap.build(RC.planar(), 20000, 0.05, 0.5, seed=3)
m.save(os.path.join(HERE, "reach_planar.sbrm"))
print("ok")
