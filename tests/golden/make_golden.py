"""Generate the golden fixtures in tests/golden/ from the reference itself.

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
Every fixture is produced by oracle/_ref/libsbref.so -- the unmodified reference sources
compiled in place plus the Appendix-C driver -- and is consumed by tests/test_golden.py
(restated oracle, CPU) and tests/test_gpu_golden.py (the CUDA path). Scenes are rebuilt from
scenes.py at test time; the stored mesh fingerprints pin that they are byte-identical.
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2512_16896_b200 import _capi as A  # noqa: E402
from paper_2512_16896_b200 import scenes  # noqa: E402
import paper_2512_16896_b200 as pkg  # noqa: E402

CACH, FALL, YAW = 0x63616368, 0x66616C6C, 0x79617721


def local_vector_scene():
    base = scenes.tabletop_boxes(32, n_objects=6, attempts=32, table=(1.6, 1.2))
    base.placements[2].relation = pkg.Relation(anchor=1, distance_type=A.SB_DIST_GREATER,
                                               direction=A.SB_DIR_FRONT, distance=0.2,
                                               angle_threshold=math.pi / 3)
    base.placements[3].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_EQUAL,
                                               direction=A.SB_DIR_VECTOR,
                                               direction_vector=(0.3, -0.4), distance=0.3,
                                               frame=A.SB_FRAME_LOCAL)
    base.placements[4].orientation = A.SB_ORIENT_FACE_TO
    base.placements[4].face_target = 0
    base.placements[5].relation = pkg.Relation(anchor=4, distance_type=A.SB_DIST_LESS,
                                               distance=0.35)
    return base


SCENES = {
    "c1_n64": lambda: scenes.tabletop_boxes(64),
    "c2_n32": lambda: scenes.tabletop_mixed(32, n_objects=9),
    "c3_n16": lambda: scenes.kitchen(16, n_objects=14, attempts=32),
    "c4_n8": lambda: scenes.dense_clutter(8, n_objects=12),
    "relations_n32": local_vector_scene,
}


def kats():
    L = O.lib()
    t = [-0.6, -0.4, 0.6, -0.4, 0.6, 0.4, -0.6, 0.4]
    jump = O.polygon_draws(t, 1, [3, CACH], 100000)
    return {
        "mix64_0": L.ref_mix64(0),
        "stream_key_1_2": L.ref_stream_key2(1, 2),
        "pcg_12345_next_u64": L.ref_pcg_next_u64(12345),
        "make_stream_7_123_double": O.stream_doubles(7, [1, 2, 3], 1)[0],
        "fast_draws_seed42": O.polygon_draws([0, 0, 1, 0, 1, 1, 0, 1], 42, [0, CACH], 3).tolist(),
        "jump_draws": {str(j): jump[j].tolist() for j in (0, 1, 7, 4095, 4096, 65535, 99999)},
        "fallback_inst1": O.polygon_draws([1, 0, 2, 0, 2, 1, 1, 1], 31, [9, FALL, 1, 7], 1)[0].tolist(),
        "fallback_inst3": O.polygon_draws([3, 0, 4, 0, 4, 1, 3, 1], 31, [9, FALL, 3, 7], 1)[0].tolist(),
        "yaw_inst1": 0.0 + (2.0 * math.pi - 0.0) * O.stream_doubles(31, [9, YAW, 1, 7], 1)[0],
        "triangulate_unit_rect": O.triangulate([0, 0, 1, 0, 1, 1, 0, 1]).tolist(),
        "region_fingerprint_unit_rect": L.ref_region_fingerprint_rect(0, 0, 1, 1),
    }


def tritri(rng):
    P = rng.uniform(-1, 1, (4000, 18))
    P[:1500, 9:] = P[:1500, :9] + rng.normal(0, 0.05, (1500, 9))
    P[1500:2500, [2, 5, 8, 11, 14, 17]] = 0.0  # coplanar pairs
    return P, O.tri_tri(P)


def world_case(rng, upright):
    meshes = [pkg.make_box(0.1, 0.08, 0.12), pkg.make_cylinder(0.05, 0.1, 16),
              scenes.sphere_set(scenes.Pcg32(99)), scenes.open_container(0.3, 0.25, 0.15, 0.01)]
    n, n_obj = 64, 6
    W = O.RefWorld(n)
    gids = [W.register_geometry(m.vertices, m.triangles) for m in meshes]
    obj_mesh, poses, enabled = [], [], []

    def pose():
        m = np.eye(4)
        if upright:
            a = rng.uniform(0, 2 * math.pi)
            m[:2, :2] = [[math.cos(a), -math.sin(a)], [math.sin(a), math.cos(a)]]
        else:
            q = rng.normal(size=4)
            w, x, y, z = q / np.linalg.norm(q)
            m[:3, :3] = [[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                         [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                         [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]]
        m[:3, 3] = rng.uniform(-0.12, 0.12, 3)
        return m

    for k in range(n_obj):
        mi = int(rng.integers(len(meshes)))
        o = W.add_object(gids[mi])
        ps = np.stack([pose() for _ in range(n)])
        W.update_transforms(o, pkg.colmajor(ps))
        en = np.nonzero(rng.random(n) < 0.75)[0].astype(np.uint32)
        W.set_enabled(o, en, True)
        obj_mesh.append(mi)
        poses.append(pkg.colmajor(ps))
        mask = np.zeros(n, np.uint8)
        mask[en] = 1
        enabled.append(mask)
    act = np.sort(rng.choice(n, 48, replace=False)).astype(np.uint32)
    cand = pkg.colmajor(np.stack([pose() for _ in act]))
    cmesh = int(rng.integers(len(meshes)))
    free, contact = W.check_batch(gids[cmesh], cand, act)
    return dict(obj_mesh=np.array(obj_mesh), poses=np.stack(poses), enabled=np.stack(enabled),
                active=act, cand=cand, cand_mesh=np.array(cmesh), free=free, contact=contact)


def main():
    O.build()
    rng = np.random.default_rng(2512)
    json.dump(kats(), open(os.path.join(HERE, "kat.json"), "w"), indent=1)
    P, r = tritri(rng)
    np.savez_compressed(os.path.join(HERE, "tritri.npz"), p=P, hit=r)
    for k, upright in enumerate([True, False, True]):
        np.savez_compressed(os.path.join(HERE, f"world{k}.npz"), **world_case(rng, upright))
    for name, make in SCENES.items():
        sc = make()
        out = O.generate(sc, 7, threads=1)
        fps = np.array([m.fingerprint() for m in sc.meshes], np.uint64)
        st = out["stats"]
        np.savez_compressed(os.path.join(HERE, f"gen_{name}.npz"), accepted=out["accepted"],
                            valid=out["valid"], poses=out["poses"], mesh_fp=fps,
                            stats=np.array([st["valid_instances"], st["candidate_checks"],
                                            st["narrow_phase_tests"], st["rounds"],
                                            st["per_instance_placements"]], np.uint64))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
