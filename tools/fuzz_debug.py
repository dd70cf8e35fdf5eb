import sys; sys.path.insert(0,'.')
import numpy as np
import importlib.util
spec=importlib.util.spec_from_file_location('f','tests/test_gpu_fuzz.py'); f=importlib.util.module_from_spec(spec); spec.loader.exec_module(f)
import paper_2512_16896_b200 as pkg
from oracle import oracle as O
for seed in [int(x) for x in sys.argv[1:]] or (16, 18):
    sc=f.random_scene(pkg, seed)
    eng=pkg.Engine(sc); got=eng.generate(seed+1); want=O.generate(sc, seed+1, threads=8)
    ref=pkg.from_colmajor(want['poses'])
    bad=~np.isclose(got.poses, ref, rtol=1e-5, atol=1e-12)
    idx=np.argwhere(bad)
    for p,i,r,c in idx:
        print(seed, 'placement', p, 'inst', i, 'entry', r, c, got.poses[p,i,r,c], ref[p,i,r,c], 'accepted', got.accepted[p,i], want['accepted'][p,i])
        print('  relation', sc.placements[p].relation, 'orient', sc.placements[p].orientation, 'face', sc.placements[p].face_target)
        print('  got', got.poses[p,i].round(6).tolist())
        print('  ref', ref[p,i].round(6).tolist())
