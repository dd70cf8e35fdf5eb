"""TEST INFRASTRUCTURE ONLY -- a pure-Python restatement of the reference hot path.

Independent of the compiled reference (oracle/_ref) and of the product: it re-derives
the reference's algorithm from /root/reference/proj (file:line cited per function) so the
two oracles check each other, and both are pinned to the committed golden fixtures
(tests/golden/, generated from oracle/_ref by tests/golden/make_golden.py).
Python floats are IEEE doubles and CPython evaluates each operation with one rounding,
so with the reference's operation order (Eigen expressions reduce left to right, see
oracle/shim/Eigen/Dense) the arithmetic is bit-identical to the -ffp-contract=off build.
`math.sin/cos/atan2` are glibc, as in the reference.

Slow by design (pure Python loops): use small N and few objects.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

M64 = (1 << 64) - 1
K_EPS = 1e-12  # collision.cpp:11
CACHE_SALT = 0x63616368  # "cach" sampler.cpp:9
FALL_SALT = 0x66616C6C   # "fall" sampler.cpp:10
YAW_SALT = 0x79617721    # "yaw!" sampler.cpp:11


# ----------------------------------------------------------------- rng.hpp:9-67
def mix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def stream_key(parts: Sequence[int]) -> int:
    h = 0x853C49E6748FEA9B
    for p in parts:
        h = mix64(h ^ p)
    return h


class Pcg32:
    MULT = 6364136223846793005

    def __init__(self, seed: int, seq: int = 0xDA3E39CB94B95BDB):
        self.state = 0
        self.inc = ((seq << 1) | 1) & M64
        self.next_u32()
        self.state = (self.state + seed) & M64
        self.next_u32()

    def next_u32(self) -> int:
        old = self.state
        self.state = (old * self.MULT + self.inc) & M64
        xs = (((old >> 18) ^ old) >> 27) & 0xFFFFFFFF
        rot = old >> 59
        return ((xs >> rot) | (xs << ((32 - rot) & 31))) & 0xFFFFFFFF

    def next_u64(self) -> int:  # GCC evaluates the left call first (rng.hpp:42)
        hi = self.next_u32()
        lo = self.next_u32()
        return (hi << 32) | lo

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()


def make_stream(seed: int, counters: Sequence[int]) -> Pcg32:
    h = mix64(seed)
    for c in counters:
        h = mix64(h ^ c)
    return Pcg32(h)


# ------------------------------------------------------------ small linear algebra
# Vectors are tuples; a pose is a 3x4 row-major tuple-of-rows [R | t] with an implicit
# bottom row (0,0,0,1) (transform.hpp; all reference poses are homogeneous).
def sub(a, b):
    return tuple(x - y for x, y in zip(a, b))


def dot(a, b):  # Eigen dot: left to right
    s = a[0] * b[0]
    for k in range(1, len(a)):
        s += a[k] * b[k]
    return s


def cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def norm(a):
    return math.sqrt(dot(a, a))


def xform(M, p):  # transform_point (transform.hpp:71-73): (R p) + t
    return tuple(((M[i][0] * p[0] + M[i][1] * p[1]) + M[i][2] * p[2]) + M[i][3] for i in range(3))


def mat_mul(A, B):  # Mat4 product rows 0..2, bottom rows (0,0,0,1) (shim order)
    out = []
    for i in range(3):
        row = []
        for j in range(4):
            b3 = 1.0 if j == 3 else 0.0
            s = A[i][0] * B[0][j]
            s = s + A[i][1] * B[1][j]
            s = s + A[i][2] * B[2][j]
            s = s + A[i][3] * b3
            row.append(s)
        out.append(tuple(row))
    return tuple(out)


def inverse_rigid(P):  # transform.hpp:63-69
    rt = [[P[k][i] for k in range(3)] for i in range(3)]
    t = (P[0][3], P[1][3], P[2][3])
    rows = []
    for i in range(3):
        s = (-rt[i][0]) * t[0]
        s = s + (-rt[i][1]) * t[1]
        s = s + (-rt[i][2]) * t[2]
        rows.append((rt[i][0], rt[i][1], rt[i][2], s))
    return tuple(rows)


def from_colmajor(c):
    return tuple(tuple(c[4 * j + i] for j in range(4)) for i in range(3))


def to_colmajor(M):
    out = [0.0] * 16
    for i in range(3):
        for j in range(4):
            out[4 * j + i] = M[i][j]
    out[15] = 1.0
    return out


# ------------------------------------------------------------------ aabb.hpp
def std_min(a, b):
    return b if b < a else a


def std_max(a, b):
    return b if a < b else a


def aabb_of(points):
    mn = [math.inf] * 3
    mx = [-math.inf] * 3
    for p in points:
        for k in range(3):
            mn[k] = std_min(mn[k], p[k])
            mx[k] = std_max(mx[k], p[k])
    return tuple(mn), tuple(mx)


def transform_aabb(M, box):  # aabb.hpp:54-62
    mn, mx = box
    c = tuple((mn[k] + mx[k]) * 0.5 for k in range(3))
    h = tuple((mx[k] - mn[k]) * 0.5 for k in range(3))
    cw = xform(M, c)
    wh = tuple((abs(M[i][0]) * h[0] + abs(M[i][1]) * h[1]) + abs(M[i][2]) * h[2] for i in range(3))
    return tuple(cw[k] - wh[k] for k in range(3)), tuple(cw[k] + wh[k] for k in range(3))


def overlaps(a, b):  # aabb.hpp:29-33, margin 0
    (amn, amx), (bmn, bmx) = a, b
    return all(amn[k] <= bmx[k] and bmn[k] <= amx[k] for k in range(3))


# ------------------------------------------------------------------ trimesh.cpp
@dataclass
class Mesh:
    v: List[Tuple[float, float, float]]
    t: List[Tuple[int, int, int]]


def make_box(sx, sy, sz):  # trimesh.cpp:40-53
    x, y, z = sx / 2, sy / 2, sz / 2
    v = [(-x, -y, -z), (x, -y, -z), (x, y, -z), (-x, y, -z),
         (-x, -y, z), (x, -y, z), (x, y, z), (-x, y, z)]
    t = [(0, 2, 1), (0, 3, 2), (4, 5, 6), (4, 6, 7), (0, 1, 5), (0, 5, 4),
         (2, 3, 7), (2, 7, 6), (1, 2, 6), (1, 6, 5), (3, 0, 4), (3, 4, 7)]
    return Mesh(v, t)


def make_sphere(radius, stacks=12, slices=16):  # trimesh.cpp:78-104
    v = [(0.0, 0.0, radius)]
    for s in range(1, stacks):
        phi = math.pi * s / stacks
        for k in range(slices):
            lam = 2.0 * math.pi * k / slices
            v.append((radius * math.sin(phi) * math.cos(lam), radius * math.sin(phi) * math.sin(lam),
                      radius * math.cos(phi)))
    south = len(v)
    v.append((0.0, 0.0, -radius))

    def ring(s, k):
        return 1 + (s - 1) * slices + (k % slices)

    t = [(0, ring(1, k), ring(1, k + 1)) for k in range(slices)]
    for s in range(1, stacks - 1):
        for k in range(slices):
            t.append((ring(s, k), ring(s + 1, k), ring(s + 1, k + 1)))
            t.append((ring(s, k), ring(s + 1, k + 1), ring(s, k + 1)))
    t += [(south, ring(stacks - 1, k + 1), ring(stacks - 1, k)) for k in range(slices)]
    return Mesh(v, t)


def drop_degenerate(m: Mesh, eps=1e-12):  # trimesh.cpp:16-29
    kept = []
    for tri in m.t:
        if any(i >= len(m.v) for i in tri):
            continue
        e1 = sub(m.v[tri[1]], m.v[tri[0]])
        e2 = sub(m.v[tri[2]], m.v[tri[0]])
        if 0.5 * norm(cross(e1, e2)) <= eps:
            continue
        kept.append(tri)
    return Mesh(list(m.v), kept)


# ------------------------------------------- libstdc++ std::nth_element (GCC 13)
# MeshBvh's leaves depend on nth_element's tie-breaking, so the restatement follows
# libstdc++'s introselect literally (bits/stl_algo.h __introselect / heap select /
# insertion sort) rather than any "equivalent" selection.
def _lg(n):
    return n.bit_length() - 1


def _adjust_heap(a, first, hole, length, value, comp):
    top = hole
    second = hole
    while second < (length - 1) // 2:
        second = 2 * (second + 1)
        if comp(a[first + second], a[first + second - 1]):
            second -= 1
        a[first + hole] = a[first + second]
        hole = second
    if (length & 1) == 0 and second == (length - 2) // 2:
        second = 2 * (second + 1)
        a[first + hole] = a[first + second - 1]
        hole = second - 1
    parent = (hole - 1) // 2
    while hole > top and comp(a[first + parent], value):
        a[first + hole] = a[first + parent]
        hole = parent
        parent = (hole - 1) // 2
    a[first + hole] = value


def _heap_select(a, first, middle, last, comp):
    length = middle - first
    if length >= 2:
        parent = (length - 2) // 2
        while True:
            _adjust_heap(a, first, parent, length, a[first + parent], comp)
            if parent == 0:
                break
            parent -= 1
    for i in range(middle, last):
        if comp(a[i], a[first]):
            value = a[i]
            a[i] = a[first]
            _adjust_heap(a, first, 0, length, value, comp)


def _move_median_to_first(a, result, x, y, z, comp):
    if comp(a[x], a[y]):
        if comp(a[y], a[z]):
            a[result], a[y] = a[y], a[result]
        elif comp(a[x], a[z]):
            a[result], a[z] = a[z], a[result]
        else:
            a[result], a[x] = a[x], a[result]
    elif comp(a[x], a[z]):
        a[result], a[x] = a[x], a[result]
    elif comp(a[y], a[z]):
        a[result], a[z] = a[z], a[result]
    else:
        a[result], a[y] = a[y], a[result]


def _unguarded_partition(a, first, last, pivot, comp):
    while True:
        while comp(a[first], a[pivot]):
            first += 1
        last -= 1
        while comp(a[pivot], a[last]):
            last -= 1
        if not first < last:
            return first
        a[first], a[last] = a[last], a[first]
        first += 1


def _insertion_sort(a, first, last, comp):
    if first == last:
        return
    for i in range(first + 1, last):
        if comp(a[i], a[first]):
            val = a[i]
            a[first + 1:i + 1] = a[first:i]
            a[first] = val
        else:
            val = a[i]
            j = i
            while comp(val, a[j - 1]):
                a[j] = a[j - 1]
                j -= 1
            a[j] = val


def nth_element(a, first, nth, last, comp):
    if first == last or nth == last:
        return
    depth = _lg(last - first) * 2
    while last - first > 3:
        if depth == 0:
            _heap_select(a, first, nth + 1, last, comp)
            a[first], a[nth] = a[nth], a[first]
            return
        depth -= 1
        mid = first + (last - first) // 2
        _move_median_to_first(a, first, first + 1, mid, last - 1, comp)
        cut = _unguarded_partition(a, first + 1, last, first, comp)
        if cut <= nth:
            first = cut
        else:
            last = cut
    _insertion_sort(a, first, last, comp)


# --------------------------------------------------------- MeshBvh (collision.cpp)
class MeshBvh:
    """collision.cpp:217-281 build; children read as {left, left+1} by collide()."""

    def __init__(self, m: Mesh):
        if not m.t:
            raise ValueError("MeshBvh: empty mesh")
        self.nodes = []  # [box, left, start, count]
        self.tris = []   # leaf-order triangle vertices
        cent = []
        for tri in m.t:
            a, b, c = (m.v[i] for i in tri)
            cent.append(tuple(((a[k] + b[k]) + c[k]) / 3.0 for k in range(3)))
        order = list(range(len(m.t)))
        self.depth = 0

        def tri_box(t):
            return aabb_of([m.v[i] for i in m.t[t]])

        def build(begin, end, depth):
            self.depth = max(self.depth, depth)
            idx = len(self.nodes)
            self.nodes.append(None)
            mn = [math.inf] * 3
            mx = [-math.inf] * 3
            for i in range(begin, end):
                tmn, tmx = tri_box(order[i])
                for k in range(3):
                    mn[k] = std_min(mn[k], tmn[k])
                    mx[k] = std_max(mx[k], tmx[k])
            box = (tuple(mn), tuple(mx))
            if end - begin <= 4:
                self.nodes[idx] = [box, -1, len(self.tris), end - begin]
                for i in range(begin, end):
                    self.tris.append(tuple(m.v[j] for j in m.t[order[i]]))
                return idx
            cmn, cmx = aabb_of([cent[order[i]] for i in range(begin, end)])
            ext = sub(cmx, cmn)
            axis = 0
            if ext[1] > ext[0]:
                axis = 1
            if ext[2] > ext[axis]:
                axis = 2
            mid = (begin + end) // 2
            nth_element(order, begin, mid, end, lambda x, y: cent[x][axis] < cent[y][axis])
            self.nodes[idx] = [box, -1, 0, 0]
            left = build(begin, mid, depth + 1)
            self.nodes[idx][1] = left
            build(mid, end, depth + 1)
            return idx

        build(0, len(m.t), 1)

    def collide(self, other: "MeshBvh", M) -> Tuple[bool, int]:
        """collision.cpp:285-329 literally (stack order, revisits, early exit)."""
        pairs = 0
        stack = [(0, 0)]
        while stack:
            a, b = stack.pop()
            na, nb = self.nodes[a], other.nodes[b]
            nb_in_a = transform_aabb(M, nb[0])
            if not overlaps(na[0], nb_in_a):
                continue
            la, lb = na[1] < 0, nb[1] < 0
            if la and lb:
                for i in range(na[2], na[2] + na[3]):
                    for j in range(nb[2], nb[2] + nb[3]):
                        q = tuple(xform(M, p) for p in other.tris[j])
                        pairs += 1
                        if tri_tri_intersect(self.tris[i], q):
                            return True, pairs
            else:
                ext_a = sub(na[0][1], na[0][0])
                ext_b = sub(nb_in_a[1], nb_in_a[0])
                if lb or (not la and dot(ext_a, ext_a) >= dot(ext_b, ext_b)):
                    stack.append((na[1], b))
                    stack.append((na[1] + 1, b))
                else:
                    stack.append((a, nb[1]))
                    stack.append((a, nb[1] + 1))
        return False, pairs


# ------------------------------------------------- tri_tri_intersect (collision.cpp)
def _isect(vv0, vv1, vv2, d0, d1, d2):  # collision.cpp:14-20
    t0 = vv0 + (vv1 - vv0) * d0 / (d0 - d1)
    t1 = vv2 + (vv1 - vv2) * d2 / (d2 - d1)
    return std_min(t0, t1), std_max(t0, t1)


def _interval(p0, p1, p2, d0, d1, d2):  # collision.cpp:23-40
    if d0 * d1 > 0.0:
        return _isect(p0, p2, p1, d0, d2, d1)
    if d0 * d2 > 0.0:
        return _isect(p0, p1, p2, d0, d1, d2)
    if d1 * d2 > 0.0 or d0 != 0.0:
        return _isect(p1, p0, p2, d1, d0, d2)
    if d1 != 0.0:
        return _isect(p0, p1, p2, d0, d1, d2)
    if d2 != 0.0:
        return _isect(p0, p2, p1, d0, d2, d1)
    return None


def _orient(p, q, r):
    return (q[0] - p[0]) * (r[1] - p[1]) - (q[1] - p[1]) * (r[0] - p[0])


def _seg_cross(a, b, c, d):  # collision.cpp:42-51
    o1, o2 = _orient(a, b, c), _orient(a, b, d)
    o3, o4 = _orient(c, d, a), _orient(c, d, b)
    return (((o1 > K_EPS and o2 < -K_EPS) or (o1 < -K_EPS and o2 > K_EPS)) and
            ((o3 > K_EPS and o4 < -K_EPS) or (o3 < -K_EPS and o4 > K_EPS)))


def _point_in_tri(p, a, b, c):  # collision.cpp:53-61
    d1, d2, d3 = _orient(a, b, p), _orient(b, c, p), _orient(c, a, p)
    neg = d1 < -K_EPS or d2 < -K_EPS or d3 < -K_EPS
    pos = d1 > K_EPS or d2 > K_EPS or d3 > K_EPS
    return not (neg and pos) and (neg or pos)


def _coplanar(n, P, Q):  # collision.cpp:63-83
    an = tuple(abs(x) for x in n)
    axis = 0
    if an[1] > an[0]:
        axis = 1
    if an[2] > an[axis]:
        axis = 2
    u, v = (axis + 1) % 3, (axis + 2) % 3
    t1 = [(p[u], p[v]) for p in P]
    t2 = [(q[u], q[v]) for q in Q]
    for i in range(3):
        for j in range(3):
            if _seg_cross(t1[i], t1[(i + 1) % 3], t2[j], t2[(j + 1) % 3]):
                return True
    c1 = (((t1[0][0] + t1[1][0]) + t1[2][0]) / 3.0, ((t1[0][1] + t1[1][1]) + t1[2][1]) / 3.0)
    c2 = (((t2[0][0] + t2[1][0]) + t2[2][0]) / 3.0, ((t2[0][1] + t2[1][1]) + t2[2][1]) / 3.0)
    return _point_in_tri(c1, *t2) or _point_in_tri(c2, *t1)


def tri_tri_intersect(P, Q) -> bool:  # collision.cpp:87-130
    p0, p1, p2 = P
    q0, q1, q2 = Q
    n2 = cross(sub(q1, q0), sub(q2, q0))
    d2c = -dot(n2, q0)
    dp = [dot(n2, p) + d2c for p in P]
    tol2 = K_EPS * std_max(1.0, norm(n2))
    dp = [0.0 if abs(x) < tol2 else x for x in dp]
    if all(x > 0 for x in dp) or all(x < 0 for x in dp):
        return False
    n1 = cross(sub(p1, p0), sub(p2, p0))
    d1c = -dot(n1, p0)
    dq = [dot(n1, q) + d1c for q in Q]
    tol1 = K_EPS * std_max(1.0, norm(n1))
    dq = [0.0 if abs(x) < tol1 else x for x in dq]
    if all(x > 0 for x in dq) or all(x < 0 for x in dq):
        return False
    if dp[0] == 0 and dp[1] == 0 and dp[2] == 0:
        return _coplanar(n1, P, Q)
    d = cross(n1, n2)
    ad = tuple(abs(x) for x in d)
    axis = 0
    if ad[1] > ad[0]:
        axis = 1
    if ad[2] > ad[axis]:
        axis = 2
    i1 = _interval(p0[axis], p1[axis], p2[axis], *dp)
    if i1 is None:
        return _coplanar(n1, P, Q)
    i2 = _interval(q0[axis], q1[axis], q2[axis], *dq)
    if i2 is None:
        return _coplanar(n1, P, Q)
    return i1[1] > i2[0] + K_EPS and i2[1] > i1[0] + K_EPS


# -------------------------------------------------- CollisionWorld (collision.cpp)
class CollisionWorld:
    """collision.cpp:334-461 for tests: objects disabled at identity until updated."""

    def __init__(self, n: int):
        self.n = n
        self.geoms = []  # (bvh, local_box)
        self.objects = []  # [geom, poses[n], boxes[n], enabled[n]]
        self.narrow = 0
        self.checked = 0

    def register_geometry(self, m: Mesh) -> int:
        m2 = drop_degenerate(m)
        self.geoms.append((MeshBvh(m2), aabb_of(m2.v)))
        return len(self.geoms) - 1

    def add_object(self, geom: int) -> int:
        ident = ((1.0, 0.0, 0.0, 0.0), (0.0, 1.0, 0.0, 0.0), (0.0, 0.0, 1.0, 0.0))
        box = self.geoms[geom][1]
        self.objects.append([geom, [ident] * self.n, [box] * self.n, [False] * self.n])
        return len(self.objects) - 1

    def update_transform(self, obj: int, inst: int, P) -> None:
        o = self.objects[obj]
        o[1][inst] = P
        o[2][inst] = transform_aabb(P, self.geoms[o[0]][1])

    def set_enabled(self, obj: int, inst: int, flag: bool) -> None:
        self.objects[obj][3][inst] = flag

    def check(self, geom: int, P, inst: int) -> int:
        """One candidate: first colliding object id or -1 (collision.cpp:433-449)."""
        bvh, local = self.geoms[geom]
        cbox = transform_aabb(P, local)
        inv = inverse_rigid(P)
        self.checked += 1
        for ob, o in enumerate(self.objects):
            if not o[3][inst] or not overlaps(cbox, o[2][inst]):
                continue
            self.narrow += 1
            hit, _ = bvh.collide(self.geoms[o[0]][0], mat_mul(inv, o[1][inst]))
            if hit:
                return ob
        return -1


# ------------------------------------------------------ polygons (polygon.cpp)
def _cross2(o, a, b):
    return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])


def ring_area(r):  # polygon.cpp:58-66
    s = 0.0
    for i in range(len(r)):
        a, b = r[i], r[(i + 1) % len(r)]
        s += a[0] * b[1] - b[0] * a[1]
    return 0.5 * s


def _in_tri_strict(p, a, b, c):
    return _cross2(a, b, p) > 1e-12 and _cross2(b, c, p) > 1e-12 and _cross2(c, a, p) > 1e-12


def ear_clip(ring) -> List[tuple]:  # polygon.cpp:260-340
    clean = []
    for p in ring:
        if clean:
            d = sub(p, clean[-1])
            if not (d[0] * d[0] + d[1] * d[1] > 1e-24):
                continue
        clean.append(p)
    while len(clean) > 1:
        d = sub(clean[0], clean[-1])
        if d[0] * d[0] + d[1] * d[1] <= 1e-24:
            clean.pop()
        else:
            break
    n = len(clean)
    out = []
    if n < 3:
        return out
    prv = [(i + n - 1) % n for i in range(n)]
    nxt = [(i + 1) % n for i in range(n)]
    reflex = [False] * n

    def upd(i):
        reflex[i] = _cross2(clean[prv[i]], clean[i], clean[nxt[i]]) < 0.0

    for i in range(n):
        upd(i)

    def is_ear(i):
        if reflex[i]:
            return False
        a, b, c = clean[prv[i]], clean[i], clean[nxt[i]]
        if abs(_cross2(a, b, c)) < 1e-18:
            return False
        j = nxt[nxt[i]]
        while j != prv[i]:
            if reflex[j] and _in_tri_strict(clean[j], a, b, c):
                return False
            j = nxt[j]
        return True

    remaining, cur, since = n, 0, 0

    def clip(k):
        p, q = prv[k], nxt[k]
        out.append((clean[p], clean[k], clean[q]))
        nxt[p] = q
        prv[q] = p
        upd(p)
        upd(q)
        return q

    while remaining > 3:
        if is_ear(cur):
            cur = clip(cur)
            remaining -= 1
            since = 0
            continue
        cur = nxt[cur]
        since += 1
        if since > remaining:
            best, best_a = -1, -1.0
            j = cur
            for _ in range(remaining):
                if not reflex[j]:
                    a = _cross2(clean[prv[j]], clean[j], clean[nxt[j]])
                    if a > best_a:
                        best_a, best = a, j
                j = nxt[j]
            if best < 0:
                break
            cur = clip(best)
            remaining -= 1
            since = 0
    if remaining == 3:
        out.append((clean[prv[cur]], clean[cur], clean[nxt[cur]]))
    return out


def triangulate(ring):  # polygon.cpp:344-368 (hole-free)
    r = list(ring)
    if len(r) < 3:
        return []
    if ring_area(r) < 0.0:
        r.reverse()
    return ear_clip(r)


class PolygonSampler:  # polygon.cpp:370-400
    def __init__(self, parts: Sequence[Sequence[tuple]]):
        self.tris, self.cum, total = [], [], 0.0
        for ring in parts:
            for t in triangulate(ring):
                a = 0.5 * abs(_cross2(*t))
                if a <= 0.0:
                    continue
                self.tris.append(t)
                total += a
                self.cum.append(total)
        if total > 0.0:
            self.cum = [c / total for c in self.cum]
            self.cum[-1] = 1.0
        else:
            self.tris, self.cum = [], []

    def valid(self) -> bool:
        return bool(self.tris)

    def draw(self, rng: Pcg32):
        u, r1, r2 = rng.next_double(), rng.next_double(), rng.next_double()
        lo, hi = 0, len(self.cum)
        while lo < hi:
            mid = (lo + hi) // 2
            if self.cum[mid] < u:
                lo = mid + 1
            else:
                hi = mid
        a, b, c = self.tris[min(len(self.tris) - 1, lo)]
        s = math.sqrt(r1)
        wa, wb, wc = 1.0 - s, s * (1.0 - r2), s * r2
        return ((a[0] * wa + b[0] * wb) + c[0] * wc, (a[1] * wa + b[1] * wb) + c[1] * wc)


def region_fingerprint(parts) -> int:  # polygon.cpp:422-444 (hole-free parts)
    h = 0x9E3779B97F4A7C15
    for ring in parts:
        h = mix64(h ^ len(ring))
        for x, y in ring:
            h = mix64(h ^ struct.unpack("<Q", struct.pack("<d", x))[0])
            h = mix64(h ^ struct.unpack("<Q", struct.pack("<d", y))[0])
    return h


class SampleCache:  # sampler.hpp:18-36, refill_cache / drain_cache (sampler.cpp:14-43)
    def __init__(self):
        self.refill_factor, self.fingerprint, self.stream = 4.0, 0, 0
        self.sampler, self.queue, self.refill_count = None, [], 0

    def bind_stream(self, key: int):
        if self.stream != key:
            self.queue = []
            self.stream = key

    def refill(self, parts, n: int, rng: Pcg32):
        fp = region_fingerprint(parts)
        if fp != self.fingerprint:
            self.queue = []
            self.sampler = PolygonSampler(parts)
            self.fingerprint = fp
        target = max(int(self.refill_factor * float(n)), n)
        if len(self.queue) >= target:
            return
        for _ in range(target - len(self.queue)):
            self.queue.append(self.sampler.draw(rng))
        self.refill_count += 1

    def drain(self, parts, k: int, rng: Pcg32):
        if region_fingerprint(parts) != self.fingerprint or len(self.queue) < k:
            self.refill(parts, max(k, 1), rng)
        out, self.queue = self.queue[:k], self.queue[k:]
        return out


class PositionSampler:  # sampler.cpp:54-127; region: list of rings or per-instance lists
    def __init__(self, salt: int):
        self.salt, self.cache = salt, SampleCache()

    def prepare(self, region, n: int, run_seed: int, per_instance: bool = False):
        self.region, self.per_instance, self.n, self.run_seed = region, per_instance, n, run_seed
        self.cache.bind_stream(stream_key([run_seed, self.salt, CACHE_SALT]))
        self.rng = make_stream(run_seed, [self.salt, CACHE_SALT])
        self.fallback = [None] * n if per_instance else []

    def sample(self, support_rows, active, attempt: int):
        """support_rows[i]: 3x4 row-major support pose of instance i."""
        pos, placeable = [(0.0, 0.0, 0.0)] * len(active), [1] * len(active)
        if not self.per_instance:
            if not self.region:
                return pos, [0] * len(active)
            pts = self.cache.drain(self.region, len(active), self.rng)
            for j, inst in enumerate(active):
                pos[j] = xform(support_rows[inst], (pts[j][0], pts[j][1], 0.0))
            return pos, placeable
        for j, inst in enumerate(active):
            reg = self.region[inst]
            if not reg:
                placeable[j] = 0
                continue
            if self.fallback[inst] is None:
                self.fallback[inst] = PolygonSampler(reg)
            if not self.fallback[inst].valid():
                placeable[j] = 0
                continue
            p = self.fallback[inst].draw(make_stream(self.run_seed, [self.salt, FALL_SALT, inst, attempt]))
            pos[j] = xform(support_rows[inst], (p[0], p[1], 0.0))
        return pos, placeable


def sample_orientations(kind: int, active, positions, face_targets, run_seed: int, salt: int,
                        attempt: int):  # sampler.cpp:129-156; kind 0 fixed, 1 uniform, 2 face_to
    yaws = [0.0] * len(active)
    for j, inst in enumerate(active):
        if kind == 1:
            yaws[j] = make_stream(run_seed, [salt, YAW_SALT, inst, attempt]).uniform(0.0, 2.0 * math.pi)
        elif kind == 2:  # face_to_yaw (relationships.cpp:232-239)
            dx = face_targets[inst][0] - positions[j][0]
            dy = face_targets[inst][1] - positions[j][1]
            yaws[j] = 0.0 if math.sqrt(dx * dx + dy * dy) < 1e-12 else math.atan2(dy, dx)
    return yaws


def rect_ring(x0, y0, x1, y1):  # make_rect (polygon.cpp:84-88)
    return [(x0, y0), (x1, y0), (x1, y1), (x0, y1)]


def annulus_sector(center, v, theta, min_r, max_r, clip_diag):  # polygon.cpp:136-176
    if not theta > 0.0 or theta > math.pi + 1e-12:
        raise ValueError("annulus_sector: theta outside (0, pi]")
    if math.isinf(max_r):
        max_r = std_max(clip_diag, min_r + 1e-6)
    if not min_r < max_r:
        raise ValueError("annulus_sector: min_r >= max_r")
    base = math.atan2(v[1], v[0])
    full = theta >= math.pi - 1e-12
    step = 5.0 * math.pi / 180.0

    def arc(radius, a0, a1, out):
        n = max(1, int(math.ceil(abs(a1 - a0) / step)))
        for i in range(n + 1):
            a = a0 + (a1 - a0) * float(i) / n
            out.append((center[0] + radius * math.cos(a), center[1] + radius * math.sin(a)))

    ext = []
    if full:
        if min_r > 0.0:
            raise ValueError("full annulus with a hole is out of scope")
        arc(max_r, 0.0, 2.0 * math.pi, ext)
        ext.pop()
        return ext
    arc(max_r, base - theta, base + theta, ext)
    if min_r > 0.0:
        arc(min_r, base + theta, base - theta, ext)
    else:
        ext.append(center)
    return ext


def clip_rect(ring, rect):
    """The oracle's Boost intersection stand-in (oracle/shim/boost/geometry.hpp)."""
    r = list(ring)
    if ring_area(r) < 0.0:  # bg::correct on the closed ring keeps vertex 0 first
        r = [r[0]] + r[:0:-1]
    x0, x1 = min(rect[0], rect[2]), max(rect[0], rect[2])
    y0, y1 = min(rect[1], rect[3]), max(rect[1], rect[3])
    for axis, bound, ge in ((0, x0, True), (0, x1, False), (1, y0, True), (1, y1, False)):
        out = []
        n = len(r)
        for i in range(n):
            cur, prv = r[i], r[(i + n - 1) % n]
            ci = cur[axis] >= bound if ge else cur[axis] <= bound
            pi = prv[axis] >= bound if ge else prv[axis] <= bound
            if ci != pi:
                o = 1 - axis
                t = (bound - prv[axis]) / (cur[axis] - prv[axis])
                val = prv[o] + t * (cur[o] - prv[o])
                out.append((bound, val) if axis == 0 else (val, bound))
            if ci:
                out.append(cur)
        r = out
    dedup = []
    for p in r:
        if not dedup or p != dedup[-1]:
            dedup.append(p)
    while len(dedup) > 1 and dedup[0] == dedup[-1]:
        dedup.pop()
    if len(dedup) < 3 or ring_area(dedup) == 0.0:
        return []
    return dedup


def relation_region(rel, rect, anchor_xy, anchor_yaw):
    """build_constraint_region's region_for(i) for one anchor (relationships.cpp:188-205)."""
    dist_t, direction, frame, dvec, d, theta = rel
    min_r, max_r = 0.0, math.inf  # distance_band (relationships.cpp:101-122)
    if dist_t == 1:
        min_r = d
    elif dist_t == 2:
        max_r = d
    elif dist_t == 3:
        half = std_max(0.05 * d, 0.01)
        min_r, max_r = std_max(0.0, d - half), d + half
    if theta <= 0:
        theta = math.pi if direction == 0 else math.pi / 4.0
    v = (1.0, 0.0)
    if direction:
        v = {1: (-1.0, 0.0), 2: (1.0, 0.0), 3: (0.0, -1.0), 4: (0.0, 1.0)}.get(direction)
        if v is None:
            nrm = math.sqrt(dvec[0] * dvec[0] + dvec[1] * dvec[1])
            v = (dvec[0] / nrm, dvec[1] / nrm)
        if frame == 1:
            c, s = math.cos(anchor_yaw), math.sin(anchor_yaw)
            v = (c * v[0] - s * v[1], s * v[0] + c * v[1])
    pts = rect_ring(*rect) + [anchor_xy]
    mn = [math.inf, math.inf]
    mx = [-math.inf, -math.inf]
    for p in pts:
        for k in range(2):
            mn[k] = std_min(mn[k], p[k])
            mx[k] = std_max(mx[k], p[k])
    dx, dy = mx[0] - mn[0], mx[1] - mn[1]
    diag = 0.0 if mn[0] > mx[0] else math.sqrt(dx * dx + dy * dy)
    ring = annulus_sector(anchor_xy, v, theta, min_r, max_r, diag)
    return clip_rect(ring, rect)


# ------------------------------------------------ the rejection loop (Appendix C)
def _rows(colmajor16):
    return from_colmajor(list(colmajor16))


def generate(scene, run_seed: int):
    """SPEC.md:516-542 with the frozen Appendix-C contract (oracle/ref_driver.cpp).

    `scene` is a paper_2512_16896_b200.world.Scene (data only). Returns a dict like
    oracle.generate: accepted [P][N], valid [N], poses [P][N][16] (column-major),
    stats {candidate_checks, narrow_phase_tests, rounds, per_instance_placements}."""
    from paper_2512_16896_b200.world import colmajor  # layout helper only

    N, K = scene.n_instances, scene.attempts
    world = CollisionWorld(N)
    meshes = [Mesh([tuple(map(float, v)) for v in m.vertices.tolist()],
                   [tuple(map(int, t)) for t in m.triangles.tolist()]) for m in scene.meshes]
    geom = [world.register_geometry(m) for m in meshes]
    for f in scene.fixed:
        obj = world.add_object(geom[f.mesh])
        P = _rows(colmajor(f.pose))
        for i in range(N):
            world.update_transform(obj, i, P)
            world.set_enabled(obj, i, True)
    pobj = [world.add_object(geom[pl.mesh]) for pl in scene.placements]
    valid = [True] * N
    accepted = [[-1] * N for _ in scene.placements]
    rounds = per_inst = 0
    for p, pl in enumerate(scene.placements):
        sup = scene.supports[pl.support]
        S = _rows(colmajor(sup.pose))
        rect = tuple(map(float, sup.rect))
        canon = rect_ring(*rect)
        if getattr(sup, "polygon", None) is not None:
            # a polygon support (e.g. from extract_support_surfaces): the ring as given feeds
            # the sampler; this restatement clips only axis-aligned rectangles (convex
            # polygons are covered by the compiled reference, tests/test_region_widening.py)
            canon = [(float(x), float(y)) for x, y in sup.polygon]
            xs, ys = [q[0] for q in canon], [q[1] for q in canon]
            rect = (min(xs), min(ys), max(xs), max(ys))
            if len(canon) != 4 or any(x not in (rect[0], rect[2]) or y not in (rect[1], rect[3])
                                      for x, y in canon):
                raise NotImplementedError("restate: non-rectangular polygon support")
        z_off = -aabb_of(meshes[pl.mesh].v)[0][2] + 1e-3  # rest_pose (sampler.cpp:45-52)
        r = pl.relation
        regions = None
        if r.anchor >= 0:
            inv_s = inverse_rigid(S)
            states = []
            for i in range(N):
                rel = mat_mul(inv_s, world.objects[pobj[r.anchor]][1][i])
                states.append(((rel[0][3], rel[1][3]), math.atan2(rel[1][0], rel[0][0])))
            spec = (r.distance_type, r.direction, r.frame, tuple(r.direction_vector),
                    r.distance, r.angle_threshold)
            vary = any(norm(sub(s[0], states[0][0])) > 1e-12 or abs(s[1] - states[0][1]) > 1e-12
                       for s in states[1:])
            if vary:
                per_inst += 1
                regions = [relation_region(spec, rect, s[0], s[1]) for s in states]
            else:
                canon = relation_region(spec, rect, states[0][0], states[0][1])
        fifo = None
        if regions is None and canon:
            fifo = (PolygonSampler([canon]), make_stream(run_seed, [p, CACHE_SALT]))
        samplers = {}
        active = [i for i in range(N) if valid[i]]
        for a in range(K):
            if not active:
                break
            rounds += 1
            nxt = []
            for i in active:
                pos = None
                if regions is None:
                    if fifo is not None:
                        x, y = fifo[0].draw(fifo[1])
                        pos = xform(S, (x, y, 0.0))
                elif regions[i]:
                    if i not in samplers:
                        samplers[i] = PolygonSampler([regions[i]])
                    if samplers[i].valid():
                        x, y = samplers[i].draw(make_stream(run_seed, [p, FALL_SALT, i, a]))
                        pos = xform(S, (x, y, 0.0))
                if pos is None:  # placeable == 0: a failed attempt (Appendix C.6)
                    nxt.append(i)
                    continue
                yaw = 0.0
                if pl.orientation == 1:
                    yaw = make_stream(run_seed, [p, YAW_SALT, i, a]).uniform(0.0, 2.0 * math.pi)
                elif pl.orientation == 2:
                    tp = world.objects[pobj[pl.face_target]][1][i]
                    d = (tp[0][3] - pos[0], tp[1][3] - pos[1])
                    yaw = 0.0 if math.sqrt(d[0] * d[0] + d[1] * d[1]) < 1e-12 else math.atan2(d[1], d[0])
                c, s = math.cos(yaw), math.sin(yaw)
                T = ((1.0, 0.0, 0.0, pos[0] + 0.0), (0.0, 1.0, 0.0, pos[1] + 0.0),
                     (0.0, 0.0, 1.0, pos[2] + z_off))
                Rz = ((c, -s, 0.0, 0.0), (s, c, 0.0, 0.0), (0.0, 0.0, 1.0, 0.0))
                P = mat_mul(T, Rz)
                if world.check(geom[pl.mesh], P, i) < 0:
                    world.update_transform(pobj[p], i, P)
                    world.set_enabled(pobj[p], i, True)
                    accepted[p][i] = a
                else:
                    nxt.append(i)
            active = nxt
        for i in active:
            valid[i] = False
    poses = [[to_colmajor(world.objects[o][1][i]) for i in range(N)] for o in pobj]
    return {"accepted": accepted, "valid": valid, "poses": poses,
            "stats": {"candidate_checks": world.checked, "narrow_phase_tests": world.narrow,
                      "rounds": rounds, "per_instance_placements": per_inst}}
