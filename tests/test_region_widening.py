"""Relation / support widening on CPU: `middle` relations over 2-8
anchors, the multi-anchor relation, convex polygon supports (incl. rectangles given as
polygons in any vertex order) and apply_ratio_on_support erosion on them.

The product's region pipeline (sb_poly.h: middle_polygon, the convex-clip stand-in,
erosion, triangulation; the code the serial region kernel runs) is restated on the host
(sb_region_draws_host) and compared with the reference's own build_constraint_region +
PolygonSampler (oracle/_ref, with the Boost stand-in of oracle/shim) by sampler draws from
the same stream: the triangle tables must agree bit for bit for the draws to."""
import math

import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A
from paper_2512_16896_b200 import world as W


def _convex_polygon(rng, k):
    """A random convex polygon with k vertices (angles sorted on an ellipse), random start
    vertex and orientation."""
    ang = np.sort(rng.uniform(0, 2 * math.pi, k))
    cx, cy = rng.uniform(-0.2, 0.2, 2)
    ax, ay = rng.uniform(0.3, 0.9, 2)
    rot = rng.uniform(0, 2 * math.pi)
    pts = np.stack([ax * np.cos(ang), ay * np.sin(ang)], 1)
    R = np.array([[math.cos(rot), -math.sin(rot)], [math.sin(rot), math.cos(rot)]])
    pts = pts @ R.T + [cx, cy]
    pts = np.roll(pts, rng.integers(k), axis=0)
    if rng.random() < 0.5:
        pts = pts[::-1]
    return pts


def _support(rng):
    kind = rng.integers(4)
    if kind == 0:
        return W.Support(np.eye(4), (-0.6, -0.4, 0.6, 0.4))
    if kind == 1:  # the same rect as a polygon, any start / orientation
        p = np.array([[-0.5, -0.35], [0.55, -0.35], [0.55, 0.45], [-0.5, 0.45]])
        p = np.roll(p, rng.integers(4), axis=0)
        return W.Support(np.eye(4), polygon=p[::-1] if rng.random() < 0.5 else p)
    if kind == 2:  # a rotated rectangle
        a = rng.uniform(0.1, 1.4)
        R = np.array([[math.cos(a), -math.sin(a)], [math.sin(a), math.cos(a)]])
        p = np.array([[-0.5, -0.3], [0.5, -0.3], [0.5, 0.3], [-0.5, 0.3]]) @ R.T
        return W.Support(np.eye(4), polygon=p)
    return W.Support(np.eye(4), polygon=_convex_polygon(rng, int(rng.integers(3, 17))))


def _relation(rng, na_max=8):
    kind = rng.integers(5)
    if kind == 0:  # middle over 2..8 anchors
        na = int(rng.integers(2, na_max + 1))
        return W.Relation(anchor=0, distance_type=A.SB_DIST_MIDDLE,
                          extra_anchors=tuple(range(1, na))), na
    if kind == 1:  # several anchors, no distance / direction: anchors[0] + full disc
        na = int(rng.integers(2, na_max + 1))
        return W.Relation(anchor=0, extra_anchors=tuple(range(1, na))), na
    dt = int(rng.choice([A.SB_DIST_NONE, A.SB_DIST_GREATER, A.SB_DIST_LESS, A.SB_DIST_EQUAL]))
    d = float(rng.uniform(0.05, 0.5))
    if kind == 2:
        return W.Relation(anchor=0, distance_type=dt, distance=d), 1
    dr = int(rng.integers(1, 6))
    return W.Relation(anchor=0, distance_type=dt, distance=d, direction=dr,
                      frame=int(rng.integers(2)),
                      direction_vector=(float(rng.uniform(-1, 1)), float(rng.uniform(-1, 1))),
                      angle_threshold=float(rng.choice([0.0, 0.3, 0.9, 1.6]))), 1


def _states(rng, na):
    s = np.zeros((na, 3))
    s[:, :2] = rng.uniform(-0.5, 0.5, (na, 2))
    s[:, 2] = rng.uniform(-math.pi, math.pi, na)
    if na >= 3 and rng.random() < 0.2:  # collinear anchors -> inflated segment
        t = rng.uniform(-1, 1, na)
        s[:, 0] = 0.1 + 0.3 * t
        s[:, 1] = -0.05 + 0.2 * t
    if na >= 3 and rng.random() < 0.15:  # two anchors on one ray from the centroid
        s[1, :2] = s[0, :2] * 1.0
    return s


def _both(ref, rel, sup, states, ratio, fx, fy, seed, c, n):
    keep = []
    r = 0.0 if ratio == 0.0 else ratio * min(fx, fy) / 2.0
    try:
        b = ref.region_draws(rel.to_c(), W.support_to_c(sup, keep), states, ratio, fx, fy, seed, c, n)
    except Exception as e:  # noqa: BLE001 -- the reference rejects it: so must we
        with pytest.raises(Exception):
            W.region_draws_host(rel, sup, states, r, seed, c, n)
        return None, str(e)
    a = W.region_draws_host(rel, sup, states, r, seed, c, n)
    return (a, b), None


def test_middle_polygon_shapes(ref):
    two = ref.middle_polygon([[0.0, 0.0], [0.4, 0.1]])
    assert two.shape == (74, 2)  # stadium: two 37-point caps
    col = ref.middle_polygon([[0.0, 0.0], [0.2, 0.1], [0.4, 0.2]])
    assert col.shape == (74, 2)
    tri = ref.middle_polygon([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    assert np.array_equal(tri, [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    same = ref.middle_polygon([[0.1, 0.1], [0.1, 0.1]])
    assert same.shape == (72, 2)  # coincident anchors: disc
    # two anchors on one ray from the centroid: the angle-sorted ring is not simple, the
    # stand-in's is_valid rejects it and the convex hull is used (ccw from lowest (x, y))
    tie = ref.middle_polygon([[0.0, 0.0], [2.0, 0.0], [1.0, 1.0], [1.5, 1.5]])
    assert len(tie) in (3, 4)


def test_region_draws_match_reference(ref):
    rng = np.random.default_rng(2512)
    checked = rejected = nonempty = 0
    for case in range(1500):
        sup = _support(rng)
        rel, na = _relation(rng)
        states = _states(rng, na)
        ratio = float(rng.choice([0.0, 0.0, 0.3, 1.0]))
        fx, fy = rng.uniform(0.02, 0.2, 2)
        res, err = _both(ref, rel, sup, states, ratio, float(fx), float(fy), 11 + case, [case, 3], 16)
        if res is None:
            rejected += 1
            continue
        (a, na_t), (b, nb_t) = res
        assert na_t == nb_t, (case, rel, sup, states)
        assert np.array_equal(a, b), (case, rel, sup, states)
        checked += 1
        nonempty += na_t > 0
    assert checked > 1200 and nonempty > 900, (checked, rejected, nonempty)


def test_no_anchor_polygon_support_regions(ref):
    """Without anchors the region is the support polygon as given (its vertex order feeds
    the triangulation); with ratio_on_support its corrected ring is eroded."""
    rng = np.random.default_rng(7)
    for case in range(200):
        sup = _support(rng)
        ratio = float(rng.choice([0.0, 0.5]))
        res, err = _both(ref, W.Relation(), sup, np.zeros((0, 3)), ratio, 0.1, 0.08, 5, [case], 24)
        assert res is not None, err
        (a, na_t), (b, nb_t) = res
        assert na_t == nb_t and np.array_equal(a, b), case


def test_relation_validation(pkg):
    sup = W.Support(np.eye(4), (-0.6, -0.4, 0.6, 0.4))
    st = np.zeros((2, 3))
    with pytest.raises(ValueError):  # middle needs >= 2 anchors
        W.region_draws_host(W.Relation(anchor=0, distance_type=A.SB_DIST_MIDDLE), sup, st[:1], 0, 1, [1], 1)
    with pytest.raises(ValueError):  # greater with two anchors
        W.region_draws_host(W.Relation(anchor=0, distance_type=A.SB_DIST_GREATER, distance=0.1,
                                       extra_anchors=(1,)), sup, st, 0, 1, [1], 1)
    with pytest.raises(ValueError):  # a direction with two anchors
        W.region_draws_host(W.Relation(anchor=0, direction=A.SB_DIR_LEFT, extra_anchors=(1,)),
                            sup, st, 0, 1, [1], 1)
    concave = W.Support(np.eye(4), polygon=[[0, 0], [1, 0], [0.2, 0.2], [0, 1]])
    with pytest.raises(ValueError):
        W.region_draws_host(W.Relation(), concave, st[:0], 0, 1, [1], 1)
