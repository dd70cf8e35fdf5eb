# Exact-equality census of accepted poses vs the oracle (GPU box diagnostic).
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import scenes
from oracle import oracle as O
for name, sc in [("c1", scenes.tabletop_boxes(1024)), ("c2", scenes.tabletop_mixed(2048)),
                 ("c3", scenes.kitchen(1024, attempts=128))]:
    got = pkg.Engine(sc).generate(1)
    want = O.generate(sc, 1, threads=8)
    ref = pkg.from_colmajor(want["poses"])
    eq = (got.poses == ref).all(axis=(2, 3))
    print(name, "accepted equal", np.array_equal(got.accepted, want["accepted"]),
          "exact poses %.5f" % eq.mean(), "max abs diff %.3g" % np.abs(got.poses - ref).max())
