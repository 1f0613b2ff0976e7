"""Closed-form pins of the oracle's frames and schedules (round-2 additions,
VERDICT r1 "What's weak" #1):

- varying XPSQ schedules (reading #8: linear from the t = 0 to the
  t = 1 value): a uniform straight spline sweeping a sphere whose radius is
  linear in t, and a cross-section plane whose (n, h) vary in t;
- the rotation convention of child-node poses in composite trees (Eqs.
  (2)-(4)): a 90-degree rotated half-box child equals the unrotated
  half-box with permuted axes, at one and at two levels of nesting;
- the constant frame of straight splines built from the up hint (reading
  #7 / #14): equals an explicitly posed SQ box minus tau ln 3;
- near-straight curved splines (1e-4 <= |A|/|B| < 1e-2, SURVEY §8(c).1 step
  8: these solve the literal cubic): brute-force projection and
  the single-root closed form phi = dist - r - tau ln 3.

Every expected value is computed here with numpy from the geometry alone
(segment projection, rotation matrices, the sphere distance), never from the
oracle's own formula."""
import math

import numpy as np
import pytest

from helpers import scene_of, pose8
from paper_2604_17538_b200 import synth

TAU_MIN = 1e-2
LN3 = math.log(3.0)


def _f(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def _eval(osc, shape, pts):
    return osc.sdf_eval(np.array([shape]), pose8().reshape(1, 8), pts, len(pts), want_pose=False)


def _segment_proj(p1, p3, x):
    B = p3 - p1
    t = ((x - p1) @ B) / B.dot(B)
    return t, p1 + np.outer(t, B)


# ---------------------------------------------------------------------------
# varying schedules (reading #8)
# ---------------------------------------------------------------------------
def test_varying_radius_straight_sphere_sweep(oracle_mod):
    """Uniform straight spline, sphere cross-section with radius r(t) = r0 +
    (r1 - r0) t: phi = |x - p(t*)| - r(t*) - tau ln 3 with t* the projection
    onto the segment (interior points).  Swapping the endpoints' radii (the
    t = 0 / t = 1 order) changes the value by (r1 - r0)(1 - 2t*)."""
    O = oracle_mod
    r0, r1 = float(np.float32(0.04)), float(np.float32(0.09))
    p1, p3 = _f([-0.3, 0.1, 0.0]), _f([0.4, -0.2, 0.1])
    ctrl = _f(np.concatenate([p1, 0.5 * (p1 + p3), p3]))
    node = synth.xpsq(ctrl=ctrl, a0=(r0, r0, r0), eps0=(1.0, 1.0), a1=(r1, r1, r1), eps1=(1.0, 1.0), up=(0, 0, 1))
    osc = O.OracleScene(scene_of([synth.make_shape("x", node)]))
    assert osc.xpsq_class(0, 0) // 10 == 1
    rng = np.random.default_rng(101)
    pts = rng.uniform(-0.5, 0.5, (600, 3))
    c = ctrl.reshape(3, 3)
    t, proj = _segment_proj(c[0], c[2], pts)
    dseg = np.linalg.norm(pts - proj, axis=1)
    ok = (t > 0.05) & (t < 0.95) & (dseg > 0.01)
    assert ok.sum() > 150
    d = _eval(osc, 0, pts[ok])["d"]
    r = r0 + (r1 - r0) * t[ok]
    assert np.allclose(d, dseg[ok] - r - TAU_MIN * LN3, atol=1e-9)
    # the reversed schedule is measurably different on these points
    r_rev = r1 + (r0 - r1) * t[ok]
    assert np.abs(d - (dseg[ok] - r_rev - TAU_MIN * LN3)).max() > 1e-2


def test_varying_plane_schedule(oracle_mod):
    """Straight spline, sphere cross-section intersected with one plane whose
    normal and offset vary linearly in t (normal renormalised, reading #8).
    Where the plane term exceeds the sphere term by > 40 tau, the smooth
    intersection equals the plane term to e^-40: phi = n(t*).y + h(t*) - tau
    ln 3, y = R^T (x - p(t*)) in the straight frame [T, b x T, b]."""
    O = oracle_mod
    r = float(np.float32(0.8))
    p1, p3 = _f([0.0, 0.0, 0.0]), _f([1.0, 0.0, 0.0])
    ctrl = _f(np.concatenate([p1, 0.5 * (p1 + p3), p3]))
    n0 = np.array([0.0, 0.0, 1.0])
    n1 = np.array([0.0, 0.6, 0.8])
    h0, h1 = -0.05, 0.02
    node = synth.xpsq(ctrl=ctrl, a0=(r, r, r), eps0=(1.0, 1.0), planes0=[[*n0, h0]], planes1=[[*n1, h1]],
                      up=(0, 0, 1))
    osc = O.OracleScene(scene_of([synth.make_shape("x", node)]))
    assert osc.xpsq_class(0, 0) // 10 == 1
    # frame: T = e_x, b = up = e_z, N = b x T = e_y
    rng = np.random.default_rng(102)
    pts = np.stack([rng.uniform(0.1, 0.9, 800), rng.uniform(-0.15, 0.15, 800), rng.uniform(0.0, 0.2, 800)], 1)
    t = pts[:, 0]
    y = np.stack([np.zeros_like(t), pts[:, 1], pts[:, 2]], 1)
    nv = (1 - t)[:, None] * _f(n0) + t[:, None] * _f(n1)
    nv /= np.linalg.norm(nv, axis=1, keepdims=True)
    h = (1 - t) * np.float32(h0) + t * np.float32(h1)
    plane = (nv * y).sum(1) + h
    sphere = np.linalg.norm(y, axis=1) - r
    ok = plane - sphere > 40 * TAU_MIN
    assert ok.sum() > 100
    d = _eval(osc, 0, pts[ok])["d"]
    assert np.allclose(d, plane[ok] - TAU_MIN * LN3, atol=1e-9)


# ---------------------------------------------------------------------------
# child-node rotation convention (Eqs. (2)-(4); node poses in the parent frame)
# ---------------------------------------------------------------------------
def _far_sphere():
    return synth.sq((0.01, 0.01, 0.01), (1.0, 1.0), pose=[5.0, 5.0, 5.0, 1, 0, 0, 0])


def _quat(axis, deg):
    return list(synth.quat_from_axis_angle(np.asarray(axis, float), math.radians(deg)))


def test_child_rotation_90z(oracle_mod):
    """union{half-box child posed at (t, +90 deg about z), far sphere} equals
    union{half-box with a_x <-> a_y swapped and the cut plane's normal e_x ->
    e_y, unrotated at t, same far sphere}: x_parent = R y_child + t, and
    R = Rz(+90) sends the child's x axis to the parent's y axis.  The
    transposed convention would put the cut on the other side (y >= 0)."""
    O = oracle_mod
    a, eps, t = (0.12, 0.05, 0.08), (0.4, 0.7), [0.03, -0.02, 0.01]
    rot = synth.op("union", [synth.psq(a, eps, [[1, 0, 0, 0.0]], pose=[*t, *_quat([0, 0, 1], 90)]), _far_sphere()])
    ref = synth.op("union", [synth.psq((a[1], a[0], a[2]), eps, [[0, 1, 0, 0.0]], pose=[*t, 1, 0, 0, 0]),
                             _far_sphere()])
    osc = O.OracleScene(scene_of([synth.make_shape("rot", rot), synth.make_shape("ref", ref)]))
    rng = np.random.default_rng(103)
    pts = np.asarray(t) + rng.uniform(-0.15, 0.15, (2000, 3))
    d_rot, d_ref = _eval(osc, 0, pts)["d"], _eval(osc, 1, pts)["d"]
    assert np.allclose(d_rot, d_ref, atol=1e-9)
    # the half-box occupies y - t_y <= 0 in the parent frame
    inside = d_rot < -1e-3
    assert inside.sum() > 20 and (pts[inside, 1] - t[1] <= 1e-3).all()


def test_child_rotation_nested(oracle_mod):
    """Two levels: a union posed at Rz(+90) containing the half-box posed at
    Rx(+90) equals the unrotated half-box with axes permuted as R = Rz Rx
    dictates (child x -> parent y, child y -> z, child z -> x), eps1 = eps2
    so every axis permutation is a symmetry of f.  The reversed composition
    Rx Rz sends child x to z instead."""
    O = oracle_mod
    a, eps = (0.12, 0.05, 0.08), (0.5, 0.5)
    inner = synth.op("union", [synth.psq(a, eps, [[1, 0, 0, 0.0]], pose=[0, 0, 0, *_quat([1, 0, 0], 90)]),
                               _far_sphere()], pose=[0, 0, 0, *_quat([0, 0, 1], 90)])
    nested = synth.op("union", [inner, synth.sq((0.01, 0.01, 0.01), (1.0, 1.0), pose=[-5.0, 5.0, 5.0, 1, 0, 0, 0])])
    # world extents: x <- a_z, y <- a_x, z <- a_y; cut plane child x <= 0 -> world y <= 0
    flat = synth.op("union", [synth.psq((a[2], a[0], a[1]), eps, [[0, 1, 0, 0.0]]), _far_sphere(),
                              synth.sq((0.01, 0.01, 0.01), (1.0, 1.0), pose=[-5.0, 5.0, 5.0, 1, 0, 0, 0])])
    osc = O.OracleScene(scene_of([synth.make_shape("n", nested), synth.make_shape("f", flat)]))
    rng = np.random.default_rng(104)
    pts = rng.uniform(-0.2, 0.2, (500, 3))
    # the outer union folds the far spheres in a different LSE nesting: both
    # are > 4 units away, weights e^-400: identical values at FP64 resolution
    assert np.allclose(_eval(osc, 0, pts)["d"], _eval(osc, 1, pts)["d"], atol=1e-9)


# ---------------------------------------------------------------------------
# straight-class constant frame from the up hint (reading #7 / #14)
# ---------------------------------------------------------------------------
def test_straight_frame_matches_posed_box(oracle_mod):
    """Straight spline along d with up hint u and an SQ box cross-section
    (a_N != a_b): for interior projections phi = SQ(R^T (x - p(t*))) - tau
    ln 3 with R = [T, b x T, b], T = d/|d|, b = Gram-Schmidt(u against T).
    The expected value is the same SQ placed explicitly with that rotation
    at p(t*) (the SQ itself is pinned in test_oracle_geometry)."""
    O = oracle_mod
    p1, p3 = _f([-0.2, 0.1, -0.1]), _f([0.3, -0.15, 0.2])
    up = _f([0.2, 0.3, 1.0])
    a, eps = (0.05, 0.04, 0.09), (0.3, 0.5)
    ctrl = _f(np.concatenate([p1, 0.5 * (p1 + p3), p3]))
    node = synth.xpsq(ctrl=ctrl, a0=a, eps0=eps, up=up)
    sc = scene_of([synth.make_shape("x", node)])
    osc = O.OracleScene(sc)
    assert osc.xpsq_class(0, 0) // 10 == 1
    T = ctrl[6:9] - ctrl[0:3]
    T /= np.linalg.norm(T)
    b = up - up.dot(T) * T
    b /= np.linalg.norm(b)
    R = np.stack([T, np.cross(b, T), b], axis=1)
    assert np.allclose(osc.xpsq_frame(0, 0, 0.3), R, atol=1e-7)
    rng = np.random.default_rng(105)
    pts = rng.uniform(-0.3, 0.3, (400, 3))
    t, proj = _segment_proj(ctrl[0:3], ctrl[6:9], pts)
    ok = (t > 0.05) & (t < 0.95) & (np.linalg.norm(pts - proj, axis=1) > 0.02)
    assert ok.sum() > 100
    d = _eval(osc, 0, pts[ok])["d"]
    # explicit posed boxes, one per point: pose (p(t*), R)
    y = np.einsum("ji,nj->ni", R, pts[ok] - proj[ok])
    expect = np.array([O.sq_phi(yy, eps, np.asarray(a, np.float32).astype(np.float64)) for yy in y])
    assert np.allclose(d, expect - TAU_MIN * LN3, atol=1e-9)
    # swapping the N and b columns (a different frame convention) is visible
    ysw = y[:, [0, 2, 1]]
    alt = np.array([O.sq_phi(yy, eps, np.asarray(a, np.float32).astype(np.float64)) for yy in ysw])
    assert np.abs(d - (alt - TAU_MIN * LN3)).max() > 1e-3


# ---------------------------------------------------------------------------
# near-straight curved splines: the literal cubic for
# 1e-4 <= |A|/|B| < 1e-2 (the survey's straight threshold is 1e-4)
# ---------------------------------------------------------------------------
def _near_straight_ctrl(ratio, rng):
    p1 = rng.uniform(-0.2, 0.2, 3)
    B = rng.normal(size=3)
    B *= 0.6 / np.linalg.norm(B)
    A = rng.normal(size=3)
    A -= A.dot(B) / B.dot(B) * B           # A perpendicular to B: a planar arc
    A *= ratio * np.linalg.norm(B) / np.linalg.norm(A)
    p2 = p1 + B / 2
    p3 = A + 2 * p2 - p1
    return _f(np.concatenate([p1, p2, p3]))


def _quad(ctrl, t):
    c = np.asarray(ctrl, dtype=np.float64).reshape(3, 3)
    t = np.asarray(t)[..., None]
    return (1 - t) ** 2 * c[0] + 2 * t * (1 - t) * c[1] + t ** 2 * c[2]


def _brute(ctrl, x, n=4001):
    ts = np.linspace(0, 1, n)
    d2 = ((_quad(ctrl, ts) - x) ** 2).sum(1)
    i = int(np.argmin(d2))
    lo, hi = ts[max(i - 1, 0)], ts[min(i + 1, n - 1)]
    f = lambda t: ((_quad(ctrl, t) - x) ** 2).sum()
    for _ in range(90):
        m1, m2 = lo + (hi - lo) * 0.381966, lo + (hi - lo) * 0.618034
        if f(m1) < f(m2):
            hi = m2
        else:
            lo = m1
    tb = 0.5 * (lo + hi)
    return tb, math.sqrt(f(tb))


@pytest.mark.parametrize("ratio", [1e-3, 5e-3, 2e-4])
def test_near_straight_projection(oracle_mod, ratio):
    """Curved class (not snapped): the root equals the brute-force (grid +
    golden-section) closest point of the quadratic to 1e-9 in t, and with a
    sphere cross-section of radius r, phi = dist - r - tau ln 3 (three
    identical roots in the one-real-root regime)."""
    O = oracle_mod
    rng = np.random.default_rng(int(ratio * 1e6))
    ctrl = _near_straight_ctrl(ratio, rng)
    r = float(np.float32(0.05))
    node = synth.xpsq(ctrl=ctrl, a0=(r, r, r), eps0=(1.0, 1.0), up=(0, 0, 1))
    osc = O.OracleScene(scene_of([synth.make_shape("x", node)]))
    assert osc.xpsq_class(0, 0) // 10 == 2, osc.xpsq_class(0, 0)
    n = 0
    for _ in range(120):
        tq = rng.uniform(0.08, 0.92)
        x = _quad(ctrl, tq) + rng.normal(size=3) * 0.08
        tb, dmin = _brute(ctrl, x)
        if not (0.02 < tb < 0.98) or dmin < 0.01:
            continue
        t, delta, wneg = osc.xpsq_roots(0, 0, x)
        assert delta < -1e3 * 1e-4 and wneg == 1.0          # one real root, far from the band
        assert np.allclose(t, tb, atol=1e-9), (t, tb)
        phi = _eval(osc, 0, x.reshape(1, 3))["d"][0]
        assert phi == pytest.approx(dmin - r - TAU_MIN * LN3, abs=1e-9)
        n += 1
    assert n > 60


def test_snap_threshold_keeps_endpoints(oracle_mod):
    """|A| < 1e-4 |B|: snapped straight onto the chord p1 -> p3 (both end
    points kept): beyond-the-end points project to t = 1 at p3 exactly."""
    O = oracle_mod
    rng = np.random.default_rng(107)
    ctrl = _near_straight_ctrl(3e-5, rng)
    r = float(np.float32(0.05))
    osc = O.OracleScene(scene_of([synth.make_shape("x", synth.xpsq(ctrl=ctrl, a0=(r, r, r), eps0=(1.0, 1.0)))]))
    assert osc.xpsq_class(0, 0) // 10 == 1
    c = ctrl.reshape(3, 3)
    e = (c[2] - c[0]) / np.linalg.norm(c[2] - c[0])
    nrm = np.cross(e, [0.3, 0.5, 0.8])
    nrm /= np.linalg.norm(nrm)
    x = c[2] + 0.2 * e + 0.01 * nrm            # beyond p3 along the chord
    t, _, _ = osc.xpsq_roots(0, 0, x)
    assert np.allclose(t, 1.0, atol=1e-12)
    phi = _eval(osc, 0, x.reshape(1, 3))["d"][0]
    assert phi == pytest.approx(np.linalg.norm(x - c[2]) - r - TAU_MIN * LN3, abs=1e-9)
