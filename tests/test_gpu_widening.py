"""GPU parity of the relation / support widening through the engine:
`middle` relations over 2-4 anchors, a multi-anchor relation, convex polygon supports
(a hexagon and a rect given as a polygon with another start vertex), ratio_on_support on
them, and sharded runs of those placements -- accepted indices, valid masks and counters
bit-exact against the reference (oracle/_ref), poses bit-identical."""
import math
import threading

import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A
from paper_2512_16896_b200 import scenes

from .test_gpu_parity import (ThreadAllgather, ThreadDevAllgather, assert_same,
                              run_generate_pair)

pytestmark = pytest.mark.gpu


def _middle_scene(pkg, n, ratio=0.0):
    base = scenes.tabletop_boxes(n, n_objects=9, table=(1.6, 1.2))
    P = base.placements
    P[3].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_MIDDLE, extra_anchors=(1,))
    P[5].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_MIDDLE, extra_anchors=(2, 4))
    P[7].relation = pkg.Relation(anchor=1, distance_type=A.SB_DIST_MIDDLE,
                                 extra_anchors=(3, 4, 6))
    P[8].relation = pkg.Relation(anchor=2, extra_anchors=(5, 6))  # multi-anchor, no distance
    if ratio:
        P[5].ratio_on_support = ratio
    return base


def _hexagon(r=0.55, rot=0.2, start=0):
    pts = [(r * math.cos(rot + k * math.pi / 3), 0.8 * r * math.sin(rot + k * math.pi / 3))
           for k in range(6)]
    return np.roll(np.array(pts), start, axis=0)


def _polygon_scene(pkg, n, clockwise=False, ratio=0.0):
    base = scenes.tabletop_boxes(n, n_objects=8, table=(1.6, 1.2))
    sup = base.supports[0]
    hexa = _hexagon(start=2)
    base.supports[0] = pkg.Support(sup.pose, polygon=hexa[::-1] if clockwise else hexa)
    # a second support: the table rect given as a polygon starting at another corner
    base.supports.append(pkg.Support(sup.pose, polygon=[[0.7, 0.5], [-0.7, 0.5], [-0.7, -0.5],
                                                        [0.7, -0.5]]))
    P = base.placements
    P[1].support = 1
    P[2].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_LESS, direction=A.SB_DIR_RIGHT,
                                 distance=0.3)
    P[3].relation = pkg.Relation(anchor=1, distance_type=A.SB_DIST_GREATER, distance=0.3)
    P[5].relation = pkg.Relation(anchor=2, distance_type=A.SB_DIST_MIDDLE, extra_anchors=(3, 4))
    P[6].support = 1
    P[6].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_EQUAL, distance=0.25)
    if ratio:
        P[0].ratio_on_support = ratio
        P[4].ratio_on_support = ratio
        P[2].ratio_on_support = ratio
    return base


@pytest.mark.parametrize("n,seed", [(1024, 3), (1, 5)])
def test_generate_middle_relations(gpu, ref, n, seed):
    eng, got, want = run_generate_pair(gpu, ref, _middle_scene(gpu, n), seed=seed)
    assert_same(gpu, got, want)


def test_generate_middle_with_ratio(gpu, ref):
    eng, got, want = run_generate_pair(gpu, ref, _middle_scene(gpu, 512, ratio=0.4), seed=9)
    assert_same(gpu, got, want)


@pytest.mark.parametrize("clockwise", [False, True])
def test_generate_polygon_supports(gpu, ref, clockwise):
    eng, got, want = run_generate_pair(gpu, ref, _polygon_scene(gpu, 1024, clockwise), seed=2)
    assert_same(gpu, got, want)
    assert got.stats["valid_instances"] > 0


def test_generate_polygon_supports_ratio(gpu, ref):
    eng, got, want = run_generate_pair(gpu, ref, _polygon_scene(gpu, 768, ratio=0.5), seed=6)
    assert_same(gpu, got, want)


def test_polygon_support_validation(gpu):
    base = scenes.tabletop_boxes(8, n_objects=2)
    base.supports[0] = gpu.Support(base.supports[0].pose,
                                   polygon=[[0, 0], [0.5, 0], [0.1, 0.1], [0, 0.5]])
    with pytest.raises(ValueError):  # not convex
        gpu.Engine(base)
    base = _middle_scene(gpu, 8)
    base.placements[3].relation = gpu.Relation(anchor=0, distance_type=A.SB_DIST_MIDDLE)
    with pytest.raises(ValueError):  # middle with one anchor
        gpu.Engine(base)
    base = _middle_scene(gpu, 8)
    base.placements[3].relation = gpu.Relation(anchor=0, distance_type=A.SB_DIST_MIDDLE,
                                               extra_anchors=(5,))
    with pytest.raises(ValueError):  # anchor after the placement
        gpu.Engine(base)


@pytest.mark.parametrize("device_exchange", [False, True])
def test_sharded_widening_equals_single(gpu, ref, device_exchange):
    """Two shards (in-process) of the middle / multi-anchor and polygon-support scenes:
    instance 0's states of every anchor travel through the exchange."""
    pkg = gpu
    for scene in (_middle_scene(pkg, 900), _polygon_scene(pkg, 700)):
        whole = pkg.Engine(scene).generate(4)
        world = 2
        ag = ThreadAllgather(world)
        agd = ThreadDevAllgather(world) if device_exchange else None
        bounds = [scene.n_instances * r // world for r in range(world + 1)]
        engines = [pkg.Engine(scene, pkg.Shard(bounds[r], bounds[r + 1], r, world, ag.fn(r),
                                               agd.fn(r) if agd else None)) for r in range(world)]
        results = [None] * world

        def run(r):
            results[r] = engines[r].generate(4)

        ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert np.array_equal(np.concatenate([r.accepted for r in results], axis=1), whole.accepted)
        assert np.array_equal(np.concatenate([r.valid for r in results]), whole.valid)
        assert np.array_equal(np.concatenate([r.poses for r in results], axis=1), whole.poses)
