"""Seeded synthetic inputs shared by the oracle, the CUDA path, the tests and
bench.py.

This module holds NO arithmetic of the method (no SDF, no projection, no
trace, no fusion): it only builds shape *descriptions* (plain parameter
dicts), static sampled-surface meshes (vertices + triangles, an input of the
method) and poses.  Meshes of superquadrics are built from the
textbook parametric superellipsoid surface (signed powers of cos/sin), not
from the paper's implicit Eq. (1).

Every float is generated in FP64 and rounded once to FP32; both the oracle
and the CUDA path consume the identical FP32 values (SURVEY §8c.1 step 9,
"input hygiene").

Configs (BASELINE.json `configs`, recipe in DESIGN.md §4):
  C1 single SQ on a plane, both directions, plus sdf_eval at 64 points
  C2 MESH box on an SQ box, parallel / slightly tilted faces, 1k envs
  C3 plane patch vs an 18-SQ smooth union, 16k envs
  C4 20 capsule-like SQ links vs a cup (cylinder (-) cylinder (+) XPSQ handle)
  C5 mixed sampled kinds x 32 SDF prototypes, 1k..1M envs
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
IDENTITY_POSE = [0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0]

# default temperatures (reading #1), per unit
# length scale ell
DEFAULT_SMOOTH = dict(tau_cmp=1e-3, tau_min=1e-2, tau_clip_alpha=1e-3, tau_clip_t=1e-3, tau_delta=1e-4,
                      trace_iters=3)


def smooth_params(ell: float = 1.0) -> dict:
    """Temperatures scaled to the scene length scale ell (lengths scale,
    dimensionless ones do not)."""
    p = dict(DEFAULT_SMOOTH)
    for k in ("tau_cmp", "tau_min", "tau_clip_alpha"):
        p[k] = float(F32(p[k] * ell))
    return p


# ---------------------------------------------------------------------------
# shape descriptions
# ---------------------------------------------------------------------------
def _f32(x):
    return [float(v) for v in np.asarray(x, dtype=np.float64).astype(F32).ravel()]


@dataclass
class Node:
    type: str
    pose: list = field(default_factory=lambda: list(IDENTITY_POSE))
    children: list = field(default_factory=list)
    eps: list = field(default_factory=lambda: [[1.0, 1.0], [1.0, 1.0]])
    a: list = field(default_factory=lambda: [[1.0, 1.0, 1.0], [1.0, 1.0, 1.0]])
    planes: list = field(default_factory=list)     # endpoint-0 rows [nx, ny, nz, h]
    planes1: list = field(default_factory=list)    # endpoint-1 rows (XPSQ)
    ctrl: list = field(default_factory=lambda: [0.0] * 9)
    up: list = field(default_factory=lambda: [0.0, 0.0, 1.0])


def _unit_rows(rows):
    out = []
    for r in rows:
        n = np.asarray(r[:3], dtype=np.float64)
        n = n / np.linalg.norm(n)
        out.append(_f32([n[0], n[1], n[2], r[3]]))
    return out


def halfspace(n, h, pose=None):
    """phi = y.n + h; inside where y.n + h <= 0."""
    return Node("halfspace", pose=_f32(pose or IDENTITY_POSE), planes=_unit_rows([[*n, h]]))


def sq(a, eps, pose=None):
    return Node("sq", pose=_f32(pose or IDENTITY_POSE), eps=[_f32(eps), _f32(eps)], a=[_f32(a), _f32(a)])


def psq(a, eps, planes, pose=None):
    return Node("psq", pose=_f32(pose or IDENTITY_POSE), eps=[_f32(eps), _f32(eps)], a=[_f32(a), _f32(a)],
                planes=_unit_rows(planes))


def xpsq(ctrl, a0, eps0, a1=None, eps1=None, planes0=(), planes1=None, up=(0.0, 0.0, 1.0), pose=None):
    a1 = a0 if a1 is None else a1
    eps1 = eps0 if eps1 is None else eps1
    planes1 = planes0 if planes1 is None else planes1
    return Node("xpsq", pose=_f32(pose or IDENTITY_POSE), eps=[_f32(eps0), _f32(eps1)], a=[_f32(a0), _f32(a1)],
                planes=_unit_rows(planes0), planes1=_unit_rows(planes1), ctrl=_f32(ctrl), up=_f32(up))


def op(kind, children, pose=None):
    assert kind in ("union", "intersection", "subtraction")
    return Node(kind, pose=_f32(pose or IDENTITY_POSE), children=list(children))


def flatten(root: Node) -> list:
    """Pre-order node list, root first; children become indices."""
    out = []

    def rec(n: Node) -> int:
        idx = len(out)
        d = dict(type=n.type, pose=list(n.pose), eps=n.eps, a=n.a, planes=n.planes, planes1=n.planes1,
                 ctrl=n.ctrl, up=n.up, children=[])
        out.append(d)
        d["children"] = [rec(c) for c in n.children]
        return idx

    rec(root)
    return out


@dataclass
class Shape:
    name: str
    sdf: list | None            # flattened node list (root first) or None
    vertices: np.ndarray | None  # [V,3] float32 local frame (sampled side)
    faces: np.ndarray | None     # [F,3] int32


def make_shape(name, root: Node | None, mesh=None) -> Shape:
    v, f = (None, None) if mesh is None else mesh
    return Shape(name, None if root is None else flatten(root),
                 None if v is None else np.ascontiguousarray(v, dtype=F32),
                 None if f is None else np.ascontiguousarray(f, dtype=np.int32))


# ---------------------------------------------------------------------------
# static sampled surfaces (inputs of the method)
# ---------------------------------------------------------------------------
def cube_grid(k: int):
    """Closed triangulated cube surface [-1,1]^3 with k x k cells per face:
    V = 6k^2 + 2, F = 12 k^2, outward winding."""
    key = {}
    verts = []

    def vid(ix, iy, iz):
        t = (ix, iy, iz)
        if t not in key:
            key[t] = len(verts)
            verts.append([2.0 * ix / k - 1.0, 2.0 * iy / k - 1.0, 2.0 * iz / k - 1.0])
        return key[t]

    faces = []
    for axis in range(3):
        for side in (0, k):
            u_ax, v_ax = [a for a in range(3) if a != axis]
            for i in range(k):
                for j in range(k):
                    q = []
                    for di, dj in ((0, 0), (1, 0), (1, 1), (0, 1)):
                        c = [0, 0, 0]
                        c[axis] = side
                        c[u_ax] = i + di
                        c[v_ax] = j + dj
                        q.append(vid(*c))
                    # orientation: outward normal along +axis when side == k
                    e1 = np.subtract(verts[q[1]], verts[q[0]])
                    e2 = np.subtract(verts[q[2]], verts[q[0]])
                    nrm = np.cross(e1, e2)
                    outward = (1.0 if side == k else -1.0)
                    if nrm[axis] * outward < 0:
                        q = q[::-1]
                    faces.append([q[0], q[1], q[2]])
                    faces.append([q[0], q[2], q[3]])
    return np.asarray(verts, dtype=np.float64), np.asarray(faces, dtype=np.int32)


def box_mesh(half, s: int):
    """Polyhedral box with half sizes `half`, each face s x s cells."""
    v, f = cube_grid(s)
    return (v * np.asarray(half, dtype=np.float64)).astype(F32), f


def _spow(x, e):
    return np.sign(x) * np.abs(x) ** e


def sq_mesh(a, eps, k: int):
    """Cube-sphere topology (k x k per face) placed on the superellipsoid
    surface by its textbook parametric form
      x = a1 C(eta)^e1 C(w)^e2, y = a2 C(eta)^e1 S(w)^e2, z = a3 S(eta)^e1
    with (eta, w) the latitude/longitude of the (tangent-warped) cube
    direction."""
    v, f = cube_grid(k)
    w = np.tan(v * (math.pi / 4.0))
    d = w / np.linalg.norm(w, axis=1, keepdims=True)
    eta = np.arcsin(np.clip(d[:, 2], -1.0, 1.0))
    om = np.arctan2(d[:, 1], d[:, 0])
    e1, e2 = eps
    ce = _spow(np.cos(eta), e1)
    p = np.stack([a[0] * ce * _spow(np.cos(om), e2), a[1] * ce * _spow(np.sin(om), e2),
                  a[2] * _spow(np.sin(eta), e1)], axis=1)
    return p.astype(F32), f


def plane_patch(n: int, m: int, sx: float, sy: float):
    """n x m vertex grid on z = 0, centred, size sx x sy; 2 triangles/cell,
    upward (+z) winding.  F = 2(n-1)(m-1)."""
    xs = np.linspace(-sx / 2, sx / 2, n)
    ys = np.linspace(-sy / 2, sy / 2, m)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    v = np.stack([X.ravel(), Y.ravel(), np.zeros(n * m)], axis=1)
    f = []
    for i in range(n - 1):
        for j in range(m - 1):
            a, b, c, d = i * m + j, (i + 1) * m + j, (i + 1) * m + j + 1, i * m + j + 1
            f.append([a, b, c])
            f.append([a, c, d])
    return v.astype(F32), np.asarray(f, dtype=np.int32)


# ---------------------------------------------------------------------------
# poses
# ---------------------------------------------------------------------------
def quat_from_axis_angle(axis, ang):
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    return np.concatenate([[math.cos(ang / 2)], math.sin(ang / 2) * axis])


def quat_mul(p, q):
    w1, x1, y1, z1 = p
    w2, x2, y2, z2 = q
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def quat_to_mat(q):
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def quats_to_mats(q):
    """Vectorised quat_to_mat over [n, 4] (w, x, y, z)."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    return np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
                     np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
                     np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], 1)


def random_quats(rng, n):
    """Uniform on SO(3) (normalised 4-D Gaussian; equivalent to the subgroup
    algorithm of)."""
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1
    return q


def pose_row(t, q):
    return np.array([t[0], t[1], t[2], q[0], q[1], q[2], q[3], 0.0])


# ---------------------------------------------------------------------------
# scenes
# ---------------------------------------------------------------------------
@dataclass
class Scene:
    name: str
    shapes: list
    smooth: dict
    pairs: np.ndarray          # [NP, 5] int32: env, slotA, slotB, shapeA (sampled), shapeB (SDF)
    poses: np.ndarray          # [n_env, n_slot, 8] float32
    ell: float = 1.0
    points: np.ndarray | None = None    # sdf_eval queries [B*P, 3]
    point_shapes: np.ndarray | None = None
    point_poses: np.ndarray | None = None  # [B, 8]
    P: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def n_env(self):
        return self.poses.shape[0]

    @property
    def n_slot(self):
        return self.poses.shape[1]

    def slice_envs(self, lo: int, hi: int) -> "Scene":
        """Env range [lo, hi) with env ids renumbered from 0 (rank shard)."""
        m = (self.pairs[:, 0] >= lo) & (self.pairs[:, 0] < hi)
        pr = self.pairs[m].copy()
        pr[:, 0] -= lo
        return Scene(self.name, self.shapes, self.smooth, np.ascontiguousarray(pr),
                     np.ascontiguousarray(self.poses[lo:hi]), self.ell, meta=dict(self.meta, env_lo=lo, env_hi=hi))


def c1_scene() -> Scene:
    """C1: SQ rounded box (a=(.20,.15,.10), eps=0.3) resting on z<=0 with
    2e-3 penetration, 2 deg tilt, 17 deg yaw; both directions; plus sdf_eval
    of the SQ at the 64 plane-patch points."""
    a, eps = (0.20, 0.15, 0.10), (0.3, 0.3)
    box = make_shape("sq_box", sq(a, eps), sq_mesh(a, eps, 3))
    ground = make_shape("ground", halfspace((0, 0, 1), 0.0), plane_patch(8, 8, 0.6, 0.6))
    q = quat_mul(quat_from_axis_angle((0, 0, 1), math.radians(17.0)),
                 quat_from_axis_angle((1, 0, 0), math.radians(2.0)))
    Rm = quat_to_mat(q)
    vz = (box.vertices.astype(np.float64) @ Rm.T)[:, 2]
    t = np.array([0.01, -0.02, -vz.min() - 2e-3])
    poses = np.zeros((1, 2, 8))
    poses[0, 0] = pose_row(t, q)
    poses[0, 1] = pose_row((0, 0, 0), (1, 0, 0, 0))
    pairs = np.array([[0, 0, 1, 0, 1], [0, 1, 0, 1, 0]], dtype=np.int32)
    sc = Scene("C1", [box, ground], smooth_params(1.0), pairs, poses.astype(F32))
    # sdf_eval: the box SDF at the 64 patch points lifted to z = 0.05
    pts = ground.vertices.astype(np.float64).copy()
    pts[:, 2] = 0.05 + 0.1 * (pts[:, 0] + 0.3)
    sc.points = pts.astype(F32)
    sc.point_shapes = np.array([0], dtype=np.int32)
    sc.point_poses = poses[0, 0:1].astype(F32)
    sc.P = 64
    return sc


def c2_scene(n_env: int = 1000, seed: int = 2) -> Scene:
    """C2: MESH box side 0.2 (6x6 per face, V=218) on an SQ box
    a=(.1,.1,.1), eps=0.1; B at origin; A at z = 0.2 - delta."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    top = make_shape("mesh_box", None, box_mesh((0.1, 0.1, 0.1), 6))
    base = make_shape("sq_box", sq((0.1, 0.1, 0.1), (0.1, 0.1)), None)
    delta = rng.uniform(0.0, 0.01, n_env)
    lat = rng.uniform(-0.05, 0.05, (n_env, 2))
    yaw = rng.uniform(0.0, 2 * math.pi, n_env)
    tilt = rng.uniform(0.0, math.radians(0.5), n_env) * (rng.uniform(size=n_env) < 0.5)
    tax = rng.uniform(0.0, 2 * math.pi, n_env)
    poses = np.zeros((n_env, 2, 8))
    for e in range(n_env):
        q = quat_mul(quat_from_axis_angle((math.cos(tax[e]), math.sin(tax[e]), 0.0), tilt[e]),
                     quat_from_axis_angle((0, 0, 1), yaw[e]))
        poses[e, 0] = pose_row((lat[e, 0], lat[e, 1], 0.2 - delta[e]), q)
        poses[e, 1] = pose_row((0, 0, 0), (1, 0, 0, 0))
    pairs = np.stack([np.arange(n_env), np.zeros(n_env), np.ones(n_env), np.zeros(n_env), np.ones(n_env)],
                     axis=1).astype(np.int32)
    return Scene("C2", [top, base], smooth_params(1.0), pairs, poses.astype(F32))


def blob18(seed: int = 3, K: int = 18):
    """Smooth union of K random SQs (the paper's 18-SQ armadillo stand-in,
    P:176)."""
    rng = np.random.Generator(np.random.Philox(key=seed + 1000))
    kids = []
    for _ in range(K):
        a = rng.uniform(0.04, 0.12, 3)
        eps = rng.uniform(0.3, 1.5, 2)
        c = rng.uniform(-0.15, 0.15, 3)
        q = random_quats(rng, 1)[0]
        kids.append(sq(a, eps, pose=[*c, *q]))
    return kids[0] if K == 1 else op("union", kids)   # a union needs >= 2 operands


def _node_surface_points(node: Node, n=400):
    """Dense parametric surface samples of the SQ leaves of a tree, in the
    tree's frame (for placing objects; input construction only)."""
    pts = []

    def rec(nd, Rp, tp):
        R = quat_to_mat(nd.pose[3:7])
        t = np.asarray(nd.pose[:3])
        Rc, tc = Rp @ R, Rp @ t + tp
        if nd.type in ("sq", "psq", "xpsq"):
            if nd.type == "xpsq":
                c = np.asarray(nd.ctrl).reshape(3, 3)
                s = np.linspace(0, 1, 20)[:, None]
                loc = (1 - s) ** 2 * c[0] + 2 * s * (1 - s) * c[1] + s ** 2 * c[2]
            else:
                v, _ = sq_mesh(nd.a[0], nd.eps[0], 8)
                loc = v.astype(np.float64)
            pts.append(loc @ Rc.T + tc)
        for ch in nd.children:
            rec(ch, Rc, tc)

    rec(node, np.eye(3), np.zeros(3))
    return np.concatenate(pts, axis=0)


def c3_scene(n_env: int = 16384, seed: int = 3, K: int = 18) -> Scene:
    """C3: 16x32 plane patch (0.4 x 0.8) sampled vs an 18-SQ smooth union."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    root = blob18(seed, K)
    surf = _node_surface_points(root)
    obj = make_shape("blob%d" % K, root, None)
    patch = make_shape("patch", None, plane_patch(16, 32, 0.4, 0.8))
    qs = random_quats(rng, n_env)
    lat = np.stack([rng.uniform(-0.1, 0.1, n_env), rng.uniform(-0.2, 0.2, n_env)], axis=1)
    pen = rng.uniform(-0.01, 0.02, n_env)
    poses = np.zeros((n_env, 2, 8))
    for e in range(n_env):
        Rm = quat_to_mat(qs[e])
        zmin = (surf @ Rm.T)[:, 2].min()
        poses[e, 0] = pose_row((0, 0, 0), (1, 0, 0, 0))
        poses[e, 1] = pose_row((lat[e, 0], lat[e, 1], -zmin - pen[e]), qs[e])
    pairs = np.stack([np.arange(n_env), np.zeros(n_env), np.ones(n_env), np.ones(n_env), np.zeros(n_env)],
                     axis=1).astype(np.int32)
    return Scene("C3", [obj, patch], smooth_params(1.0), pairs, poses.astype(F32))


def cup() -> Node:
    """Cup (Fig. 3): (outer cylinder (-) inner cylinder) (+) handle
    swept along a quadratic spline."""
    outer = sq((0.04, 0.04, 0.05), (0.1, 1.0))
    inner = sq((0.035, 0.035, 0.05), (0.1, 1.0), pose=[0, 0, 0.006, 1, 0, 0, 0])
    handle = xpsq(ctrl=[0.04, 0, 0.03, 0.075, 0, 0, 0.04, 0, -0.03], a0=(0.004, 0.006, 0.004), eps0=(0.2, 0.2),
                  up=(0, 1, 0))
    return op("union", [op("subtraction", [outer, inner]), handle])


def c4_scene(n_env: int = 65536, seed: int = 4, n_links: int = 20) -> Scene:
    """C4: 20 capsule-like SQ links (cube-sphere k=3) vs a cup, ell = 0.04."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    cup_root = cup()
    surf = _node_surface_points(cup_root)
    shapes = [make_shape("cup", cup_root, None)]
    link_a = []
    for i in range(n_links):
        lr = np.random.Generator(np.random.Philox(key=seed + 100 + i))
        a = (float(lr.uniform(0.008, 0.012)),) * 2 + (float(lr.uniform(0.02, 0.03)),)
        e1 = float(lr.uniform(0.5, 1.0))
        shapes.append(make_shape("link%d" % i, sq(a, (e1, 1.0)), sq_mesh(a, (e1, 1.0), 3)))
        link_a.append(a)
    yaw = rng.uniform(0, 2 * math.pi, n_env)
    # one shell placement per (env, link)
    dirs = rng.standard_normal((n_env, n_links, 3))
    dirs /= np.linalg.norm(dirs, axis=2, keepdims=True)
    clr = rng.uniform(-0.004, 0.006, (n_env, n_links))
    lq = random_quats(rng, n_env * n_links).reshape(n_env, n_links, 4)
    poses = np.zeros((n_env, n_links + 1, 8))
    # object surface support distance along each direction (from samples):
    # support of the yawed cup along u = support of the cup along R(yaw)^T u
    cy, sy = np.cos(yaw), np.sin(yaw)
    qo = np.stack([np.cos(yaw / 2), np.zeros(n_env), np.zeros(n_env), np.sin(yaw / 2)], 1)
    ul = np.stack([cy[:, None] * dirs[..., 0] + sy[:, None] * dirs[..., 1],
                   -sy[:, None] * dirs[..., 0] + cy[:, None] * dirs[..., 1], dirs[..., 2]], axis=-1)
    sup = np.empty((n_env, n_links))
    for lo in range(0, n_env, 4096):
        sup[lo:lo + 4096] = (ul[lo:lo + 4096] @ surf.T).max(axis=2)
    r = sup + clr + np.array([a[0] for a in link_a])[None, :]
    poses[:, 0, 3:7] = qo
    poses[:, 1:, :3] = dirs * r[..., None]
    poses[:, 1:, 3:7] = lq
    pairs = np.stack([np.repeat(np.arange(n_env), n_links), np.tile(np.arange(1, n_links + 1), n_env),
                      np.zeros(n_env * n_links), np.tile(np.arange(1, n_links + 1), n_env),
                      np.zeros(n_env * n_links)], axis=1).astype(np.int32)
    return Scene("C4", shapes, smooth_params(0.04), pairs, poses.astype(F32), ell=0.04)


def random_points(rng, n, lo, hi):
    return rng.uniform(lo, hi, (n, 3)).astype(F32)


# ---------------------------------------------------------------------------
# C5: mixed sampled kinds x 32 SDF prototypes
# ---------------------------------------------------------------------------
def psq_mesh(a, eps, planes, k: int):
    """Cube-sphere SQ mesh whose vertices outside a half-space are pulled
    radially (towards the centre, which is inside every plane) onto the
    plane: an input surface for the PSQ (star-shaped about its centre)."""
    v, f = sq_mesh(a, eps, k)
    v = v.astype(np.float64)
    for pl in planes:
        n = np.asarray(pl[:3], dtype=np.float64)
        n = n / np.linalg.norm(n)
        h = float(pl[3])
        s = v @ n
        out = s + h > 0
        v[out] *= (-h / s[out])[:, None]
    return v.astype(F32), f


def xpsq_mesh(ctrl, a, eps2, nt: int, nth: int):
    """Tube around the quadratic spline: nt rings of nth points on the
    cross-section superellipse (a_y, a_z, exponent eps2) in the Frenet frame,
    plus the two end-cap centres: V = nt nth + 2."""
    c = np.asarray(ctrl, dtype=np.float64).reshape(3, 3)
    A, B = c[0] - 2 * c[1] + c[2], 2 * (c[1] - c[0])
    b = np.cross(B, A)
    b = b / np.linalg.norm(b)
    ts = np.linspace(0.0, 1.0, nt)
    th = np.linspace(0.0, 2 * math.pi, nth, endpoint=False)
    verts = []
    for t in ts:
        p = c[0] + B * t + A * t * t
        T = B + 2 * A * t
        T = T / np.linalg.norm(T)
        N = np.cross(b, T)
        for w in th:
            verts.append(p + a[1] * _spow(math.cos(w), eps2) * N + a[2] * _spow(math.sin(w), eps2) * b)
    verts.append(c[0] - a[0] * (B / np.linalg.norm(B)))
    pe = c[0] + B + A
    Te = (B + 2 * A) / np.linalg.norm(B + 2 * A)
    verts.append(pe + a[0] * Te)
    V = len(verts)
    faces = []
    for i in range(nt - 1):
        for j in range(nth):
            a0, a1 = i * nth + j, i * nth + (j + 1) % nth
            b0, b1 = a0 + nth, a1 + nth
            faces += [[a0, b0, b1], [a0, b1, a1]]
    for j in range(nth):
        faces.append([V - 2, (j + 1) % nth, j])
        o = (nt - 1) * nth
        faces.append([V - 1, o + j, o + (j + 1) % nth])
    return np.asarray(verts, dtype=F32), np.asarray(faces, dtype=np.int32)


def _fib_dirs(n=256):
    i = np.arange(n) + 0.5
    phi = np.arccos(1 - 2 * i / n)
    th = math.pi * (1 + 5 ** 0.5) * i
    return np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], 1)


def _support_table(points, dirs):
    return (dirs @ np.asarray(points, dtype=np.float64).T).max(axis=1)


def c5_library(seed: int = 5):
    """16 sampled prototypes (spheres, MESH boxes, SQs, PSQs, curved XPSQs;
    k = 3 or 4: V = 56 or 98) and 32 SDF prototypes (4 spheres, 4 boxes, 8
    SQs, 6 PSQs, 6 curved XPSQs, 2 cups, 2 four-SQ blobs); lengths ~0.1."""
    rng = np.random.Generator(np.random.Philox(key=seed + 2000))
    sampled, sdf = [], []
    for i in range(16):
        kind = ["sphere", "box", "sq", "psq", "xpsq"][i % 5]
        k = 3 if i % 2 == 0 else 4
        if kind == "sphere":
            r = float(rng.uniform(0.03, 0.06))
            sampled.append(make_shape("s_sph%d" % i, None, sq_mesh((r, r, r), (1, 1), k)))
        elif kind == "box":
            h = rng.uniform(0.03, 0.06, 3)
            sampled.append(make_shape("s_box%d" % i, None, box_mesh(h, k)))
        elif kind == "sq":
            a, e = rng.uniform(0.03, 0.07, 3), rng.uniform(0.3, 1.5, 2)
            sampled.append(make_shape("s_sq%d" % i, None, sq_mesh(a, e, k)))
        elif kind == "psq":
            a, e = rng.uniform(0.04, 0.07, 3), rng.uniform(0.4, 1.2, 2)
            pls = [[*rng.normal(size=3), -float(rng.uniform(0.01, 0.03))] for _ in range(int(rng.integers(1, 5)))]
            sampled.append(make_shape("s_psq%d" % i, None, psq_mesh(a, e, pls, k)))
        else:
            ctrl = [-0.05, 0, 0, 0.0, 0.06, 0.0, 0.05, 0, 0.01]
            a = (0.015, 0.02, 0.015)
            nt, nth = (9, 6) if k == 3 else (12, 8)
            sampled.append(make_shape("s_xpsq%d" % i, None, xpsq_mesh(ctrl, a, 0.5, nt, nth)))
    for i in range(4):
        r = float(rng.uniform(0.03, 0.07))
        sdf.append(make_shape("sph%d" % i, sq((r, r, r), (1, 1))))
    for i in range(4):
        sdf.append(make_shape("box%d" % i, sq(rng.uniform(0.03, 0.07, 3), (0.1, 0.1))))
    for i in range(8):
        sdf.append(make_shape("sq%d" % i, sq(rng.uniform(0.03, 0.07, 3), rng.uniform(0.2, 1.8, 2))))
    for i in range(6):
        pls = [[*rng.normal(size=3), -float(rng.uniform(0.01, 0.03))] for _ in range(int(rng.integers(1, 5)))]
        sdf.append(make_shape("psq%d" % i, psq(rng.uniform(0.04, 0.07, 3), rng.uniform(0.3, 1.5, 2), pls)))
    for i in range(6):
        p1 = rng.uniform(-0.06, -0.03, 3) * [1, 0.3, 0.3]
        p3 = rng.uniform(0.03, 0.06, 3) * [1, 0.3, 0.3]
        p2 = 0.5 * (p1 + p3) + rng.uniform(0.03, 0.06) * np.array([0, 1, 0.2])
        sdf.append(make_shape("xpsq%d" % i, xpsq(np.concatenate([p1, p2, p3]), rng.uniform(0.01, 0.02, 3),
                                                  rng.uniform(0.3, 1.0, 2))))
    for i in range(2):
        sdf.append(make_shape("cup%d" % i, cup()))
    for i in range(2):
        r2 = np.random.Generator(np.random.Philox(key=seed + 3000 + i))
        kids = [sq(r2.uniform(0.015, 0.035, 3), r2.uniform(0.3, 1.5, 2),
                   pose=[*r2.uniform(-0.04, 0.04, 3), *random_quats(r2, 1)[0]]) for _ in range(4)]
        sdf.append(make_shape("blob4_%d" % i, op("union", kids)))
    return sampled, sdf


def _sdf_surface_samples(shape: Shape):
    # dense samples of the SDF prototype's constituents, for placement only
    root_nodes = shape.sdf
    pts = []

    def rec(k, R, t):
        n = root_nodes[k]
        Rc = R @ quat_to_mat(n["pose"][3:7])
        tc = R @ np.asarray(n["pose"][:3]) + t
        if n["type"] in ("sq", "psq"):
            v, _ = sq_mesh(n["a"][0], n["eps"][0], 6)
            pts.append(v.astype(np.float64) @ Rc.T + tc)
        elif n["type"] == "xpsq":
            v, _ = xpsq_mesh(n["ctrl"], n["a"][0], 0.5, 16, 8)
            pts.append(v.astype(np.float64) @ Rc.T + tc)
        for c in n["children"]:
            rec(c, Rc, tc)

    rec(0, np.eye(3), np.zeros(3))
    return np.concatenate(pts)


C5_BLOCK = 65536


def c5_scene(n_env: int = 1 << 20, env_lo: int = 0, seed: int = 5) -> Scene:
    """C5: one pair per env, uniform over (16 sampled x 32 SDF prototypes);
    B at the origin with a uniform rotation, A on a random direction with a
    support-gap clearance U[-0.025, 0.005] (about half the pairs have a
    penetrating candidate);
    ell = 0.1.  Envs [env_lo, env_lo + n_env) of a global sequence whose
    random numbers are drawn per block of 65536 envs keyed by (seed, block),
    so any rank can generate its own shard."""
    sampled, sdf = c5_library(seed)
    shapes = sampled + sdf
    dirs = _fib_dirs(512)
    supA = np.stack([_support_table(s.vertices, dirs) for s in sampled])
    supB = np.stack([_support_table(_sdf_surface_samples(s), dirs) for s in sdf])
    n_s = len(sampled)
    poses = np.zeros((n_env, 2, 8))
    pairs = np.zeros((n_env, 5), np.int32)
    e = env_lo
    while e < env_lo + n_env:
        blk = e // C5_BLOCK
        lo, hi = blk * C5_BLOCK, (blk + 1) * C5_BLOCK
        rng = np.random.Generator(np.random.Philox(key=[seed, blk]))
        ia = rng.integers(0, n_s, C5_BLOCK)
        ib = rng.integers(0, len(sdf), C5_BLOCK)
        qa = random_quats(rng, C5_BLOCK)
        qb = random_quats(rng, C5_BLOCK)
        u = rng.standard_normal((C5_BLOCK, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        clr = rng.uniform(-0.025, 0.005, C5_BLOCK)
        s, t = max(e, lo), min(env_lo + n_env, hi)
        sl = slice(s - lo, t - lo)
        # support of B along u (B rotated by qb) and of A along -u (A rotated by qa)
        Rb = quats_to_mats(qb[sl])
        Ra = quats_to_mats(qa[sl])
        ub = np.einsum("nji,nj->ni", Rb, u[sl])
        ua = np.einsum("nji,nj->ni", Ra, -u[sl])
        hb = supB[ib[sl], np.argmax(ub @ dirs.T, axis=1)]
        ha = supA[ia[sl], np.argmax(ua @ dirs.T, axis=1)]
        dist = ha + hb + clr[sl]
        o = slice(s - env_lo, t - env_lo)
        poses[o, 0, :3] = u[sl] * dist[:, None]
        poses[o, 0, 3:7] = qa[sl]
        poses[o, 1, 3:7] = qb[sl]
        pairs[o, 0] = np.arange(s - env_lo, t - env_lo)
        pairs[o, 1] = 0
        pairs[o, 2] = 1
        pairs[o, 3] = ia[sl]
        pairs[o, 4] = n_s + ib[sl]
        e = t
    return Scene("C5", shapes, smooth_params(0.1), pairs, poses.astype(F32), ell=0.1,
                 meta=dict(env_lo=env_lo, n_sampled=n_s, n_sdf=len(sdf)))


def c6_parts(seed: int, K: int = 18):
    """The K SQ parts of blob18(seed) as separate shapes: each with its SDF
    (the SQ with its part pose as node pose) and its sampled surface (the
    cube-sphere SQ mesh, k = 3, moved by the part pose): the SQ-pair
    decomposition of the paper's efficiency experiment."""
    rng = np.random.Generator(np.random.Philox(key=seed + 1000))
    parts = []
    for i in range(K):
        a = rng.uniform(0.04, 0.12, 3)
        eps = rng.uniform(0.3, 1.5, 2)
        c = rng.uniform(-0.15, 0.15, 3)
        q = random_quats(rng, 1)[0]
        v, f = sq_mesh(_f32(a), _f32(eps), 3)
        R = quat_to_mat(np.asarray(_f32(q), np.float64))
        vw = (v.astype(np.float64) @ R.T + np.asarray(_f32(c), np.float64)).astype(F32)
        parts.append(make_shape("part%d_%d" % (seed, i), sq(a, eps, pose=[*c, *q]), (vw, f)))
    return parts


def c6_scene(n_env: int = 1024, env_lo: int = 0, seed: int = 7, K: int = 18) -> Scene:
    """C6 (broad-phase workload; the paper's efficiency
    experiment P:188-201): two objects of K = 18 SQ parts each (blob18 seeds
    3 and 11); every env pairs every part of A (sampled) with every part of B
    (SDF): K^2 = 324 pairs.  B at the origin, A uniformly rotated at a
    distance U[0.15, 0.45] along a random direction (the objects' parts
    reach ~0.25 from their centres), so some part pairs touch and most are
    far apart -- the case a broad phase filters.  ell = 0.1."""
    A, B = c6_parts(3, K), c6_parts(11, K)
    shapes = A + B
    poses = np.zeros((n_env, 2, 8))
    e = env_lo
    blk_pairs = []
    while e < env_lo + n_env:
        blk = e // C5_BLOCK
        lo, hi = blk * C5_BLOCK, (blk + 1) * C5_BLOCK
        rng = np.random.Generator(np.random.Philox(key=[seed, blk]))
        qa = random_quats(rng, C5_BLOCK)
        qb = random_quats(rng, C5_BLOCK)
        u = rng.standard_normal((C5_BLOCK, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        dist = rng.uniform(0.15, 0.45, C5_BLOCK)
        s_, t_ = max(e, lo), min(env_lo + n_env, hi)
        sl = slice(s_ - lo, t_ - lo)
        o = slice(s_ - env_lo, t_ - env_lo)
        poses[o, 0, :3] = u[sl] * dist[sl, None]
        poses[o, 0, 3:7] = qa[sl]
        poses[o, 1, 3:7] = qb[sl]
        e = t_
    ia, ib = np.meshgrid(np.arange(K), np.arange(K), indexing="ij")
    per_env = np.stack([np.zeros(K * K), np.zeros(K * K), np.ones(K * K), ia.ravel(), K + ib.ravel()], 1)
    pairs = np.tile(per_env, (n_env, 1)).astype(np.int32)
    pairs[:, 0] = np.repeat(np.arange(n_env), K * K)
    return Scene("C6", shapes, smooth_params(0.1), np.ascontiguousarray(pairs), poses.astype(F32), ell=0.1,
                 meta=dict(env_lo=env_lo, parts=K))


def sdf_scene(n_body: int = 1 << 16, P: int = 64, env_lo: int = 0, seed: int = 6) -> Scene:
    """sdf_eval workload (SURVEY §8d secondary metric): the 32 C5 SDF
    prototypes, one body per batch item with a uniform rotation and a
    translation U[-0.1, 0.1]^3, and P query points per body: samples of the
    body's constituent surfaces (_sdf_surface_samples) jittered by N(0, 0.01^2)
    per axis in the body frame, then moved to world.  Bodies
    [env_lo, env_lo + n_body) of a global sequence keyed per block of 65536
    bodies (rank shards, as c5_scene)."""
    _, sdf = c5_library(5)
    surf = [_sdf_surface_samples(s) for s in sdf]
    shape_ids = np.zeros(n_body, np.int32)
    poses = np.zeros((n_body, 8))
    pts = np.zeros((n_body, P, 3))
    e = env_lo
    while e < env_lo + n_body:
        blk = e // C5_BLOCK
        lo, hi = blk * C5_BLOCK, (blk + 1) * C5_BLOCK
        rng = np.random.Generator(np.random.Philox(key=[seed, blk]))
        ib = rng.integers(0, len(sdf), C5_BLOCK)
        q = random_quats(rng, C5_BLOCK)
        t = rng.uniform(-0.1, 0.1, (C5_BLOCK, 3))
        u = rng.random((C5_BLOCK, P))
        jit = rng.normal(0.0, 0.01, (C5_BLOCK, P, 3))
        s, t_ = max(e, lo), min(env_lo + n_body, hi)
        sl, o = slice(s - lo, t_ - lo), slice(s - env_lo, t_ - env_lo)
        shape_ids[o] = ib[sl]
        poses[o, :3] = t[sl]
        poses[o, 3:7] = q[sl]
        loc = np.zeros((t_ - s, P, 3))
        for k in range(len(sdf)):
            m = ib[sl] == k
            if m.any():
                idx = np.minimum((u[sl][m] * len(surf[k])).astype(np.int64), len(surf[k]) - 1)
                loc[m] = surf[k][idx]
        loc += jit[sl]
        R = quats_to_mats(q[sl])
        pts[o] = np.einsum("nij,npj->npi", R, loc) + t[sl][:, None, :]
        e = t_
    sc = Scene("SDF", sdf, smooth_params(0.1), np.zeros((0, 5), np.int32), poses[:, None, :].astype(F32), ell=0.1,
               meta=dict(env_lo=env_lo))
    sc.points = pts.reshape(-1, 3).astype(F32)
    sc.point_shapes = shape_ids
    sc.point_poses = poses.astype(F32)
    sc.P = P
    return sc
