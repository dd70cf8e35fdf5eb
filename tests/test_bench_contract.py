"""bench.py's reference arm (CPU): the reference runs alone in its process (only
oracle/_ref/libsbref.so mapped), on a scene built with the reference's own mesh
constructors that is byte-identical to the product's, with the same `config` object."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config", ["c1_tabletop", "c2_mixed", "c3_kitchen", "c4_clutter",
                                    "c5_sweep100"])
def test_reference_scene_is_byte_identical(config, ref):
    sys.path.insert(0, ROOT)
    import bench

    class Args:
        pass

    a = Args()
    a.config, a.n = config, 0
    mine = bench.WORKLOADS[config][1](32)
    theirs = bench.reference_scene(a, 32)
    assert len(mine.meshes) == len(theirs.meshes)
    for m1, m2 in zip(mine.meshes, theirs.meshes):
        assert np.array_equal(m1.vertices, m2.vertices)
        assert np.array_equal(m1.triangles, m2.triangles)
    assert bench.workload_config(a, 1, mine) == bench.workload_config(a, 1, theirs)


def test_reference_arm_maps_only_the_reference(ref):
    code = (
        "import json, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c2_mixed', "
        "'--ref-n', '64', '--steps', '1', '--warmup', '0']; import bench; bench.main(); "
        "maps = sorted({l.split()[-1] for l in open('/proc/self/maps') if l.rstrip().endswith('.so')});"
        " print(json.dumps(maps))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=600, check=True).stdout.strip().splitlines()
    line = json.loads(out[0])
    maps = json.loads(out[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["n_instances_per_gpu"] == 16384
    mine = [m for m in maps if os.path.abspath(m).startswith(ROOT)]
    assert mine == [os.path.join(ROOT, "oracle", "_ref", "libsbref.so")], mine
