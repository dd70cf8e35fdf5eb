"""CPU: pin both oracles to the golden fixtures generated from the reference itself
(tests/golden/make_golden.py, from oracle/_ref). The pure-Python restatement
(oracle/restate.py) must reproduce every fixture bit for bit; so must the compiled
reference when it is present."""
import json
import math
import os

import numpy as np
import pytest

from oracle import restate as R
from paper_2512_16896_b200 import scenes

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCENE_NAMES = ["c1_n64", "c2_n32", "c3_n16", "c4_n8", "relations_n32"]


def scene(name):
    import importlib.util

    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(GOLD, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    return mg.SCENES[name]()


def test_kat_fixture_matches_survey_appendix_a():
    k = json.load(open(os.path.join(GOLD, "kat.json")))
    assert k["mix64_0"] == 0xE220A8397B1DCDAF
    assert k["stream_key_1_2"] == 0xE39317DCDF18B70D
    assert k["pcg_12345_next_u64"] == 0x8630B53A16AC2A2C
    assert k["make_stream_7_123_double"] == 0.31432417967541759
    assert k["jump_draws"]["4095"] == [0.3617226090254968, 0.39531144032076443]
    assert k["jump_draws"]["99999"] == [-0.41236551912179142, -0.22015113274073267]
    assert k["fallback_inst3"] == [3.4801327803400239, 0.50989079180751684]
    assert k["yaw_inst1"] == 5.9471590821050837
    assert k["region_fingerprint_unit_rect"] == 0x5B65160753483216


def test_restated_rng_and_sampler_match_kats():
    k = json.load(open(os.path.join(GOLD, "kat.json")))
    assert R.mix64(0) == k["mix64_0"]
    assert R.stream_key([1, 2]) == k["stream_key_1_2"]
    assert R.Pcg32(12345).next_u64() == k["pcg_12345_next_u64"]
    assert R.make_stream(7, [1, 2, 3]).next_double() == k["make_stream_7_123_double"]
    s = R.PolygonSampler([R.rect_ring(0, 0, 1, 1)])
    rng = R.make_stream(42, [0, R.CACHE_SALT])
    assert [list(s.draw(rng)) for _ in range(3)] == k["fast_draws_seed42"]
    table = R.PolygonSampler([R.rect_ring(-0.6, -0.4, 0.6, 0.4)])
    rng = R.make_stream(1, [3, R.CACHE_SALT])
    draws = [table.draw(rng) for _ in range(4097)]
    for j in ("0", "1", "7", "4095", "4096"):
        assert list(draws[int(j)]) == k["jump_draws"][j]
    f = R.PolygonSampler([R.rect_ring(3, 0, 4, 1)]).draw(R.make_stream(31, [9, R.FALL_SALT, 3, 7]))
    assert list(f) == k["fallback_inst3"]
    y = R.make_stream(31, [9, R.YAW_SALT, 1, 7]).uniform(0.0, 2.0 * math.pi)
    assert y == k["yaw_inst1"]
    tris = [[list(p) for p in t] for t in R.triangulate(R.rect_ring(0, 0, 1, 1))]
    assert tris == k["triangulate_unit_rect"]


def test_restated_tri_tri_matches_fixture():
    g = np.load(os.path.join(GOLD, "tritri.npz"))
    P, hit = g["p"], g["hit"]
    got = [R.tri_tri_intersect([tuple(p[0:3]), tuple(p[3:6]), tuple(p[6:9])],
                               [tuple(p[9:12]), tuple(p[12:15]), tuple(p[15:18])]) for p in P]
    assert np.array_equal(np.array(got, np.uint8), hit)
    assert 0.2 < hit.mean() < 0.8


def _world_meshes():
    import paper_2512_16896_b200 as pkg

    return [pkg.make_box(0.1, 0.08, 0.12), pkg.make_cylinder(0.05, 0.1, 16),
            scenes.sphere_set(scenes.Pcg32(99)), scenes.open_container(0.3, 0.25, 0.15, 0.01)]


@pytest.mark.parametrize("k", [0, 1, 2])
def test_restated_check_batch_matches_fixture(k):
    g = np.load(os.path.join(GOLD, f"world{k}.npz"))
    meshes = _world_meshes()
    n = g["poses"].shape[1]
    W = R.CollisionWorld(n)
    gids = [W.register_geometry(R.Mesh([tuple(v) for v in m.vertices.tolist()],
                                       [tuple(t) for t in m.triangles.tolist()])) for m in meshes]
    for o, mi in enumerate(g["obj_mesh"]):
        W.add_object(gids[int(mi)])
        for i in range(n):
            W.update_transform(o, i, R.from_colmajor(list(g["poses"][o, i])))
            W.set_enabled(o, i, bool(g["enabled"][o, i]))
    free = np.ones(n, np.uint8)
    contact = np.full(n, -1, np.int32)
    for j, inst in enumerate(g["active"]):
        c = W.check(gids[int(g["cand_mesh"])], R.from_colmajor(list(g["cand"][j])), int(inst))
        if c >= 0:
            free[inst], contact[inst] = 0, c
    assert np.array_equal(free, g["free"]) and np.array_equal(contact, g["contact"])


@pytest.mark.parametrize("name", SCENE_NAMES)
def test_scenes_reproduce_fixture_meshes(name):
    g = np.load(os.path.join(GOLD, f"gen_{name}.npz"))
    fps = np.array([m.fingerprint() for m in scene(name).meshes], np.uint64)
    assert np.array_equal(fps, g["mesh_fp"])


@pytest.mark.parametrize("name", ["c2_n32", "c3_n16", "c4_n8", "relations_n32"])
def test_restated_generation_matches_fixture(name):
    g = np.load(os.path.join(GOLD, f"gen_{name}.npz"))
    r = R.generate(scene(name), 7)
    assert np.array_equal(np.array(r["accepted"], np.int16), g["accepted"])
    assert np.array_equal(np.array(r["valid"], np.uint8), g["valid"])
    assert np.array_equal(np.array(r["poses"]), g["poses"])  # bit-exact: same libm (glibc)
    st = r["stats"]
    assert [st["candidate_checks"], st["narrow_phase_tests"], st["rounds"],
            st["per_instance_placements"]] == [int(x) for x in g["stats"][1:]]


@pytest.mark.parametrize("name", SCENE_NAMES)
def test_compiled_reference_matches_fixture(ref, name):
    g = np.load(os.path.join(GOLD, f"gen_{name}.npz"))
    r = ref.generate(scene(name), 7, threads=4)
    assert np.array_equal(r["accepted"], g["accepted"])
    assert np.array_equal(r["valid"], g["valid"])
    assert np.array_equal(r["poses"], g["poses"])
