"""Per-instance support frames and fixed-object batches (support_world[inst],
sampler.hpp:78-80 / sampler.cpp:90,119; TransformBatch fixed poses, collision.hpp:95):

* stacking -- a support on an earlier placed object: frame = its accepted pose * surface
  frame, per instance and run;
* a drawer -- a cabinet with a prismatic drawer whose per-instance joint values go through
  BatchedSceneGraph forward kinematics (scene_graph.cpp:126-147) into the drawer body's
  fixed poses and the drawer floor's support frames; a relation anchored inside the drawer.
The engine against the reference driver: accepted indices, valid masks, counters and
accepted poses bit-exact."""
import math

import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A
from paper_2512_16896_b200 import scenes
from tests.test_gpu_parity import assert_same, run_generate_pair

pytestmark = pytest.mark.gpu


def stacking_scene(pkg, n, seed=3):
    """A 0.3 x 0.25 x 0.08 crate on the table, then boxes on the crate's top (its frame:
    rotated with the crate's sampled yaw), then more boxes on the table."""
    rng = scenes.Pcg32(seed)
    base = scenes.tabletop_boxes(n, n_objects=0, table=(1.2, 0.8))
    crate = pkg.make_box(0.3, 0.25, 0.08)
    base.meshes.append(crate)
    base.placements.append(pkg.Placement(mesh=len(base.meshes) - 1, support=0))
    top = pkg.Support(pkg.translation(0.0, 0.0, 0.04), (-0.15, -0.125, 0.15, 0.125), on_placement=0)
    base.supports.append(top)
    for k in range(5):
        base.meshes.append(pkg.make_box(rng.uniform(0.03, 0.07), rng.uniform(0.03, 0.07),
                                        rng.uniform(0.03, 0.07)))
        base.placements.append(pkg.Placement(mesh=len(base.meshes) - 1, support=1 if k < 3 else 0))
    base.placements[3].relation = pkg.Relation(anchor=1, distance_type=A.SB_DIST_LESS,
                                               distance=0.12)
    return base


@pytest.mark.parametrize("n", [1, 257, 4096])
def test_stacking_on_a_placed_object(gpu, ref, n):
    scene = stacking_scene(gpu, n)
    eng, got, want = run_generate_pair(gpu, ref, scene, seed=5)
    assert_same(gpu, got, want)
    if n > 1:
        assert got.valid.sum() > 0
        # the stacked boxes rest on the crate's top: z = crate z + 0.04 + their rest offset
        ok = (got.accepted[0] >= 0) & (got.accepted[1] >= 0)
        crate_z = got.poses[0][ok][:, 2, 3]
        z1 = got.poses[1][ok][:, 2, 3]
        assert np.all(z1 > crate_z + 0.04)


def drawer_scene(pkg, n, seed=11):
    """Cabinet body (fixed) + drawer (fixed, per-instance pose from FK of a prismatic joint)
    with objects placed on the drawer floor (support frames = FK of the floor node)."""
    rng = np.random.default_rng(seed)
    g = pkg.BatchedSceneGraph(n)
    cab = g.add_node(0, "cabinet")
    g.set_edge_batch(0, cab, np.tile(pkg.translation(0.0, 1.0, 0.0), (n, 1, 1)))
    drawer = g.add_node(cab, "drawer", -1, pkg.JointSpec(1, (0.0, -1.0, 0.0), 0.0, 0.35))
    g.set_joint_states(drawer, rng.uniform(0.0, 0.35, n))
    floor = g.add_node(drawer, "floor")
    g.set_edge_batch(drawer, floor, np.tile(pkg.translation(0.0, 0.0, 0.02), (n, 1, 1)))
    drawer_world = g.world_poses(drawer)      # FK: cabinet edge * joint motion
    floor_world = g.world_poses(floor)        # ... * floor edge (the surface frame)

    base = scenes.tabletop_boxes(n, n_objects=0, table=(1.2, 0.8))
    body = scenes.open_container(0.5, 0.45, 0.3, 0.02)
    base.meshes.append(body)
    base.fixed.append(pkg.Fixed(len(base.meshes) - 1, pkg.translation(0.0, 1.0, 0.4)))
    tray = scenes.open_container(0.44, 0.4, 0.12, 0.01)
    base.meshes.append(tray)
    base.fixed.append(pkg.Fixed(len(base.meshes) - 1, np.eye(4), poses=drawer_world))
    base.supports.append(pkg.Support(np.eye(4), (-0.2, -0.18, 0.2, 0.18), poses=floor_world))
    prng = scenes.Pcg32(seed)
    for k in range(6):
        base.meshes.append(pkg.make_box(prng.uniform(0.03, 0.08), prng.uniform(0.03, 0.08),
                                        prng.uniform(0.02, 0.06)))
        base.placements.append(pkg.Placement(mesh=len(base.meshes) - 1, support=1 if k < 4 else 0))
    base.placements[2].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_LESS,
                                               distance=0.15, direction=A.SB_DIR_RIGHT)
    base.placements[3].orientation = A.SB_ORIENT_FACE_TO
    base.placements[3].face_target = 1
    return base, drawer_world


@pytest.mark.parametrize("n", [1, 300, 2048])
def test_drawer_support_from_fk(gpu, ref, n):
    scene, drawer_world = drawer_scene(gpu, n)
    eng, got, want = run_generate_pair(gpu, ref, scene, seed=2)
    assert_same(gpu, got, want)
    # objects in the drawer move with it: their y follows the per-instance drawer opening
    ok = got.accepted[0] >= 0
    if ok.sum() > 1:
        dy = got.poses[0][ok][:, 1, 3] - drawer_world[ok][:, 1, 3]
        assert np.all(np.abs(dy) <= 0.2 + 1e-9)


def test_per_instance_support_validation(gpu):
    pkg = gpu
    scene = stacking_scene(pkg, 8)
    scene.supports[1].on_placement = 1  # its own placement is not earlier
    scene.placements[1].support = 1
    with pytest.raises(ValueError):
        pkg.Engine(scene)
    scene = stacking_scene(pkg, 8)
    scene.supports[1].on_placement = -1
    scene.supports[1].poses = np.tile(np.eye(4), (7, 1, 1))  # wrong batch size
    with pytest.raises(ValueError):
        pkg.Engine(scene)
