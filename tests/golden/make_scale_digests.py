"""Reference digests for the BASELINE configs too large to re-run on every GPU test.

Run in the build container (needs oracle/_ref, i.e. /root/reference to build it):
    python tests/golden/make_scale_digests.py [name ...]
Each entry runs the reference's rejection loop (oracle/_ref/libsbref.so: the unmodified
reference sources plus the Appendix-C driver) on the full-size scene from scenes.py with
ThreadPool(nproc), and stores into tests/golden/scale_digests.json:
  * sha256 of the accepted attempt indices (int16, placement-major) and of the valid mask,
  * the reference's work counters,
  * sha256 of all accepted poses (column-major doubles; -1 placements hold whatever the
    reference driver leaves there, so the GPU test compares only the sample below),
  * a seeded sample of (placement, instance) accepted poses in scale_<name>.npz.
tests/test_gpu_scale_digests.py recomputes the same digests from the CUDA engine.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2512_16896_b200 import scenes  # noqa: E402

OUT = os.path.join(HERE, "scale_digests.json")
POSE_SAMPLES = 1024

CASES = {
    # BASELINE C5: {10, 50, 100} objects x 2^20 variations (the 10-object point is also
    # compared live in test_generate_matches_reference_at_scale)
    "c5_1M_x50": lambda: scenes.scale_sweep(1 << 20, 50),
    "c5_1M_x100": lambda: scenes.scale_sweep(1 << 20, 100),
    "c5_1M_x10": lambda: scenes.scale_sweep(1 << 20, 10),
    # C5's 100-object sweep at the smaller sizes
    "c5_64k_x100": lambda: scenes.scale_sweep(1 << 16, 100),
    "c5_1k_x100": lambda: scenes.scale_sweep(1 << 10, 100),
}


def sample_index(P: int, n: int, seed: int = 12345):
    rng = np.random.default_rng(seed)
    return rng.integers(0, P, POSE_SAMPLES), rng.integers(0, n, POSE_SAMPLES)


def digest(accepted: np.ndarray, valid: np.ndarray) -> dict:
    return {"accepted_sha256": hashlib.sha256(np.ascontiguousarray(accepted, np.int16).tobytes()).hexdigest(),
            "valid_sha256": hashlib.sha256(np.ascontiguousarray(valid, np.uint8).tobytes()).hexdigest()}


def main(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    threads = os.cpu_count() or 8
    for name in names:
        scene = CASES[name]()
        P, n = len(scene.placements), scene.n_instances
        t0 = time.time()
        r = O.generate(scene, 1, threads=threads, with_poses=True)
        dt = time.time() - t0
        pi, ii = sample_index(P, n)
        poses = r["poses"][pi, ii]  # (S, 16) column-major
        entry = {"n": n, "placements": P, "run_seed": 1, "threads": threads,
                 "ref_seconds": round(dt, 1), "stats": r["stats"],
                 "valid_count": int(r["valid"].sum()),
                 "accepted_hist": np.bincount(r["accepted"].ravel() + 1).tolist()[:8],
                 "pose_sample_seed": 12345,
                 "poses_sha256": hashlib.sha256(np.ascontiguousarray(r["poses"]).tobytes()).hexdigest()}
        entry.update(digest(r["accepted"], r["valid"]))
        np.savez_compressed(os.path.join(HERE, f"scale_{name}.npz"), poses=poses)
        data[name] = entry
        del r
        json.dump(data, open(OUT, "w"), indent=1)
        print(f"{name}: {dt:.1f} s, valid {entry['valid_count']}/{n}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
