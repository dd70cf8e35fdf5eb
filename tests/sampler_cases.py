"""Shared PositionSampler / sample_orientations scenarios (sampler.cpp:14-156) for the
oracle cross-check (CPU) and the device parity tests (GPU). Each scenario is a list of
ops run against an adapter, so the same FIFO-cache history (refills, re-prepare with the
same / a new seed, region change, m = 0, full and ragged active sets) hits every
implementation."""
import math

import numpy as np

RECT = [(-0.6, -0.4), (0.6, -0.4), (0.6, 0.4), (-0.6, 0.4)]
# concave L given clockwise (triangulate reverses it), plus a detached triangle
L_CW = [(0.0, 0.0), (0.0, 0.5), (0.2, 0.5), (0.2, 0.2), (0.6, 0.2), (0.6, 0.0)]
TRI = [(-0.5, -0.5), (-0.1, -0.45), (-0.3, -0.1)]
SLIVER = [(0.0, 0.0), (1.0, 0.0), (2.0, 0.0)]  # zero area: contributes no triangle
REGIONS = {"rect": [RECT], "lt": [L_CW, TRI], "rect+sliver": [RECT, SLIVER], "empty": []}


def supports(n, seed, upright=True):
    """(n, 4, 4) support poses (rigid)."""
    rng = np.random.default_rng(seed)
    out = np.tile(np.eye(4), (n, 1, 1))
    for i in range(n):
        if upright:
            a = rng.uniform(0, 2 * math.pi)
            out[i, :2, :2] = [[math.cos(a), -math.sin(a)], [math.sin(a), math.cos(a)]]
        else:
            q = rng.normal(size=4)
            w, x, y, z = q / np.linalg.norm(q)
            out[i, :3, :3] = [[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                              [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                              [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]]
        out[i, :3, 3] = rng.uniform(-2, 2, size=3)
    return out


def fifo_ops(n, seed):
    """prepare / sample history over canonical regions exercising every cache branch."""
    rng = np.random.default_rng(seed)

    def sub(frac):
        k = int(round(frac * n))
        return np.sort(rng.choice(n, size=k, replace=False)).astype(np.uint32)

    full = np.arange(n, dtype=np.uint32)
    return [
        ("prepare", "rect", 7), ("sample", full, 0), ("sample", sub(0.5), 1),
        ("sample", sub(0.3), 2), ("sample", sub(0.0), 3), ("sample", full, 4),
        ("sample", full, 5),                                # queue short -> refill
        ("prepare", "rect", 7), ("sample", sub(0.2), 0),    # same stream: queue kept, rng restarts
        ("sample", full, 1),
        ("prepare", "rect+sliver", 7), ("sample", sub(0.4), 0),  # new fingerprint -> queue cleared
        ("prepare", "lt", 11), ("sample", full, 0), ("sample", sub(0.7), 1),  # new seed
        ("prepare", "empty", 11), ("sample", sub(0.5), 0),  # empty region: not placeable, cache untouched
        ("prepare", "lt", 11), ("sample", sub(0.9), 0), ("sample", sub(0.05), 1),
        ("sample", full, 2), ("sample", full, 3),  # refill on top of leftover points
    ]


def per_instance_regions(n, seed):
    """One region per instance: rect / L+tri / empty / zero-area sliver, scaled per instance."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        kind = rng.integers(6)
        s = float(rng.uniform(0.5, 1.5))
        if kind == 4:
            out.append([])
        elif kind == 5:
            out.append([SLIVER])
        elif kind % 2 == 0:
            out.append([[(x * s, y * s) for x, y in RECT]])
        else:
            out.append([[(x * s, y * s) for x, y in L_CW], TRI])
    return out


def run_fifo(adapter, n, seed, support):
    """Returns [(positions, placeable, refill_count), ...] per sample op."""
    res = []
    for op in fifo_ops(n, seed):
        if op[0] == "prepare":
            adapter.prepare(REGIONS[op[1]], n, op[2], False)
        else:
            pos, pl = adapter.sample(support, op[1], op[2])
            res.append((np.asarray(pos, np.float64).reshape(-1, 3), np.asarray(pl, np.uint8),
                        adapter.refills()))
    return res


class RefAdapter:
    """oracle/_ref (the reference's PositionSampler compiled from /root/reference)."""

    def __init__(self, ref, salt):
        self.ref, self.s, self.n = ref, ref.RefSampler(salt), 0
        self.last = 0

    def prepare(self, region, n, seed, per_instance):
        if per_instance:
            rings, inst = [], [0]
            for r in region:
                rings.extend(r)
                inst.append(len(rings))
            self.s.prepare(rings, n, seed, np.asarray(inst, np.uint32))
        else:
            self.s.prepare(region, n, seed)

    def sample(self, support, active, attempt):
        cm = np.ascontiguousarray(np.swapaxes(support, -1, -2)).reshape(-1, 16)
        pos, pl, self.last = self.s.sample(cm, active, attempt)
        return pos, pl

    def refills(self):
        return self.last


class RestateAdapter:
    """oracle/restate.py (pure-Python restatement)."""

    def __init__(self, R, salt):
        self.R, self.s = R, R.PositionSampler(salt)

    def prepare(self, region, n, seed, per_instance):
        self.s.prepare(region, n, seed, per_instance)

    def sample(self, support, active, attempt):
        rows = [tuple(tuple(support[i, r, :]) for r in range(3)) for i in range(len(support))]
        return self.s.sample(rows, [int(a) for a in active], attempt)

    def refills(self):
        return self.s.cache.refill_count


class DeviceAdapter:
    """The product: sb_sampler_* through the C ABI."""

    def __init__(self, pkg, salt):
        self.s = pkg.PositionSampler(salt)

    def prepare(self, region, n, seed, per_instance):
        self.s.prepare(region, n, seed, per_instance)

    def sample(self, support, active, attempt):
        return self.s.sample(support, active, attempt)

    def refills(self):
        return self.s.cache_info()[1]
