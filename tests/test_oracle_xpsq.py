"""Pins of the oracle's XPSQ (§II-B.4, Eq. (5)-(6)):
worked cubic examples (SURVEY App. B / S:319-329), brute-force projection,
degenerate splines that reduce to closed forms, the Frenet frame, continuity
across Delta = 0, finite differences, and the cup vs a hard-boolean
membership test."""
import math

import numpy as np
import pytest

from helpers import scene_of, pose8, unpack_sym3
from paper_2604_17538_b200 import synth

TAU_MIN = 1e-2


def _xscene(O, ctrl, a=(0.05, 0.05, 0.05), eps=(1.0, 1.0), up=(0, 0, 1), **kw):
    node = synth.xpsq(ctrl=ctrl, a0=a, eps0=eps, up=up, **kw)
    sc = scene_of([synth.make_shape("x", node)])
    return O.OracleScene(sc)


def _f(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def test_arch_projection_example(oracle_mod):
    """S:328 / App. B: p1=(0,0,0), p2=(1,1,0), p3=(2,0,0), x=(1,2,0):
    c = (-8, 12, -16, 6), P = 1.25, q = 0, Delta = -7.8125, t* = 0.5."""
    osc = _xscene(oracle_mod, [0, 0, 0, 1, 1, 0, 2, 0, 0])
    t, delta, wneg = osc.xpsq_roots(0, 0, [1, 2, 0])
    assert delta == pytest.approx(-7.8125, rel=1e-12)
    assert wneg == 1.0
    assert np.allclose(t, 0.5, atol=1e-12)
    # tangent at t = 0.5 is horizontal
    R = osc.xpsq_frame(0, 0, 0.5)
    assert np.allclose(R[:, 0], [1, 0, 0], atol=1e-12)


def test_one_real_root_example(oracle_mod):
    """(t - 1/2)(t^2 + 1): Delta = -6.25, unique root 1/2.  Built from
    A = (1,0,0), B = (-1/3, sqrt(17)/3, 0), w = (0, 3/sqrt(17), 0) so that the
    monic projection cubic is t^3 - t^2/2 + t - 1/2."""
    by = math.sqrt(17.0) / 3.0
    A = np.array([1.0, 0, 0])
    B = np.array([-1.0 / 3.0, by, 0])
    p1 = np.zeros(3)
    p2 = p1 + B / 2
    p3 = A + 2 * p2 - p1
    x = p1 + np.array([0, 1.0 / by, 0])
    osc = _xscene(oracle_mod, np.concatenate([p1, p2, p3]))
    # control points are FP32-rounded: compare with a loose tolerance
    t, delta, wneg = osc.xpsq_roots(0, 0, x)
    assert delta == pytest.approx(-6.25, rel=1e-5)
    assert np.allclose(t, 0.5, atol=1e-6)


def test_three_real_roots_example(oracle_mod):
    """Roots {0.2, 0.5, 0.8} (App. B): A = (1,0,0), B = (-1,1,0),
    w = (0.34, 0.5, 0) gives the monic cubic (t-.2)(t-.5)(t-.8); Delta =
    0.002916 and the trigonometric form returns (.8, .2, .5) for k = 0,1,2."""
    osc = _xscene(oracle_mod, [0, 0, 0, -0.5, 0.5, 0, 0, 1, 0])
    t, delta, wneg = osc.xpsq_roots(0, 0, [0.34, 0.5, 0.0])
    assert delta == pytest.approx(0.002916, rel=1e-5)
    assert wneg < 1e-12
    assert np.allclose(t, [0.8, 0.2, 0.5], atol=1e-5)


def _quad(ctrl, t):
    c = np.asarray(ctrl, dtype=np.float64).reshape(3, 3)
    t = np.asarray(t)[..., None]
    return (1 - t) ** 2 * c[0] + 2 * t * (1 - t) * c[1] + t ** 2 * c[2]


def _brute_t(ctrl, x, n=20001):
    ts = np.linspace(0, 1, n)
    d2 = ((_quad(ctrl, ts) - x) ** 2).sum(1)
    i = int(np.argmin(d2))
    # local refinement by golden-section on the bracket
    lo, hi = ts[max(i - 1, 0)], ts[min(i + 1, n - 1)]
    f = lambda t: ((_quad(ctrl, t) - x) ** 2).sum()
    for _ in range(80):
        m1, m2 = lo + (hi - lo) * 0.382, lo + (hi - lo) * 0.618
        if f(m1) < f(m2):
            hi = m2
        else:
            lo = m1
    tb = 0.5 * (lo + hi)
    return tb, math.sqrt(f(tb))


def test_projection_brute_force(oracle_mod):
    """S:343 / S:659: for random curved splines and points with |Delta| >
    20 tau_Delta, the best of the three t* reaches the brute-force (grid +
    refinement) minimum distance to within 1e-3 (relative to the spline
    size)."""
    rng = np.random.default_rng(11)
    n_ok = 0
    for trial in range(300):
        ctrl = _f(rng.uniform(-1, 1, 9))
        osc = _xscene(oracle_mod, ctrl)
        if osc.xpsq_class(0, 0) != 21:
            continue
        x = rng.uniform(-1.5, 1.5, 3)
        t, delta, _ = osc.xpsq_roots(0, 0, x)
        if abs(delta) < 20 * 1e-4:
            continue
        _, dmin = _brute_t(ctrl, x)
        dk = np.sqrt(((_quad(ctrl, t) - x) ** 2).sum(1))
        assert dk.min() - dmin < 1e-3 * max(1.0, dmin), (trial, t, delta)
        n_ok += 1
    assert n_ok > 200


def test_point_spline_reduces_to_psq(oracle_mod):
    """p1 = p2 = p3 = c: exactly PSQ(x - c) - tau ln 3 (App. B)."""
    O = oracle_mod
    c = [0.1, -0.2, 0.05]
    a, eps, planes = (0.2, 0.1, 0.15), (0.7, 0.4), [[0, 0, 1, -0.05]]
    x = synth.xpsq(ctrl=c * 3, a0=a, eps0=eps, planes0=planes, up=(0, 0, 1))
    p = synth.psq(a, eps, planes, pose=[*c, 1, 0, 0, 0])
    sc = scene_of([synth.make_shape("x", x), synth.make_shape("p", p)])
    osc = O.OracleScene(sc)
    rng = np.random.default_rng(12)
    pts = rng.uniform(-0.5, 0.5, (200, 3))
    dx = osc.sdf_eval(np.array([0]), pose8().reshape(1, 8), pts, len(pts), want_pose=False)
    dp = osc.sdf_eval(np.array([1]), pose8().reshape(1, 8), pts, len(pts), want_pose=False)
    assert np.allclose(dx["d"], dp["d"] - TAU_MIN * math.log(3.0), atol=1e-12)
    assert np.allclose(dx["grad"], dp["grad"], atol=1e-12)


def test_straight_spline_capsule(oracle_mod):
    """Uniform straight spline sweeping a sphere of radius r: exactly
    (distance to the segment - r) - tau ln 3 where the closest point is
    interior (App. B)."""
    O = oracle_mod
    r = float(np.float32(0.07))
    p1, p3 = np.array([-0.3, 0.1, 0.0]), np.array([0.4, -0.2, 0.1])
    ctrl = _f(np.concatenate([p1, 0.5 * (p1 + p3), p3]))
    osc = _xscene(O, ctrl, a=(r, r, r), eps=(1.0, 1.0), up=(0, 0, 1))
    assert osc.xpsq_class(0, 0) // 10 == 1
    rng = np.random.default_rng(13)
    pts = rng.uniform(-0.5, 0.5, (400, 3))
    out = osc.sdf_eval(np.array([0]), pose8().reshape(1, 8), pts, len(pts), want_pose=False)
    c = ctrl.reshape(3, 3)
    B = 2 * (c[1] - c[0])
    t = ((pts - c[0]) @ B) / B.dot(B)
    m = (t > 0.05) & (t < 0.95)
    dseg = np.linalg.norm(pts - (c[0] + np.outer(t, B)), axis=1)
    ok = m & (dseg > 0.01)
    assert ok.sum() > 100
    assert np.allclose(out["d"][ok], dseg[ok] - r - TAU_MIN * math.log(3.0), atol=1e-9)


def test_curved_swept_sphere_bounds(oracle_mod):
    """Curved spline + sphere cross-section: phi - (brute-force distance - r)
    lies in [-tau ln 3, 0] when |Delta| >> tau_Delta (App. B)."""
    O = oracle_mod
    r = float(np.float32(0.05))
    ctrl = _f([0.0, 0.0, 0.0, 0.3, 0.4, 0.0, 0.6, -0.1, 0.2])
    osc = _xscene(O, ctrl, a=(r, r, r), eps=(1.0, 1.0))
    rng = np.random.default_rng(14)
    n = 0
    for _ in range(300):
        x = rng.uniform(-0.3, 0.9, 3)
        t, delta, _ = osc.xpsq_roots(0, 0, x)
        if abs(delta) < 20 * 1e-4:
            continue
        _, dmin = _brute_t(ctrl, x)
        if dmin < 1e-2:
            continue
        phi = osc.sdf_eval(np.array([0]), pose8().reshape(1, 8), x.reshape(1, 3), 1, want_pose=False)["d"][0]
        e = phi - (dmin - r)
        assert -TAU_MIN * math.log(3.0) - 1e-6 <= e <= 1e-6, (x, e)
        n += 1
    assert n > 150


def test_frenet_frame_properties(oracle_mod):
    rng = np.random.default_rng(15)
    for _ in range(50):
        ctrl = _f(rng.uniform(-1, 1, 9))
        osc = _xscene(oracle_mod, ctrl)
        for t in rng.uniform(0, 1, 5):
            R = osc.xpsq_frame(0, 0, t)
            assert np.allclose(R.T @ R, np.eye(3), atol=1e-12)
            assert np.linalg.det(R) == pytest.approx(1.0, abs=1e-12)
            if osc.xpsq_class(0, 0) == 21:
                c = ctrl.reshape(3, 3)
                A, B = c[0] - 2 * c[1] + c[2], 2 * (c[1] - c[0])
                pd = B + 2 * A * t
                assert np.allclose(R[:, 0], pd / np.linalg.norm(pd), atol=1e-12)
                # osculating plane: binormal is B x A direction
                bxa = np.cross(B, A)
                assert np.allclose(R[:, 2], bxa / np.linalg.norm(bxa), atol=1e-12)


def test_branch_continuity_across_delta_zero(oracle_mod):
    """a probe line that drives Delta through 0; the blended
    SDF has no jump: step-to-step increments <= 10 x the sweep step."""
    O = oracle_mod
    ctrl = _f([0, 0, 0, 1, 1, 0, 2, 0, 0])
    osc = _xscene(O, ctrl, a=(0.1, 0.1, 0.1), eps=(1.0, 1.0))
    # x moves along the symmetry axis x = 1 from above the curvature centre
    ys = np.linspace(-2.0, 0.3, 23001)
    pts = np.stack([np.full_like(ys, 1.0), ys, np.zeros_like(ys)], axis=1)
    d = osc.sdf_eval(np.array([0]), pose8().reshape(1, 8), pts, len(pts), want_pose=False)["d"]
    deltas = np.array([osc.xpsq_roots(0, 0, p)[1] for p in pts[::50]])
    assert deltas.min() < -10 * 1e-4 and deltas.max() > 10 * 1e-4, "probe must cross Delta = 0"
    step = ys[1] - ys[0]
    assert np.abs(np.diff(d)).max() <= 10 * step


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_xpsq_gradient_hessian_fd(oracle_mod, seed):
    """Jet derivatives of the XPSQ (with varying schedules and planes) vs
    central finite differences, away from |Delta| < 40 tau_Delta."""
    O = oracle_mod
    rng = np.random.default_rng(30 + seed)
    ctrl = _f(rng.uniform(-0.2, 0.2, 9))
    node = synth.xpsq(ctrl=ctrl, a0=(0.05, 0.04, 0.03), eps0=(0.5, 0.8), a1=(0.03, 0.05, 0.04), eps1=(0.9, 0.4),
                      planes0=[[0, 0, 1, -0.01]], planes1=[[0, 1, 1, -0.005]], up=(0, 0, 1))
    osc = O.OracleScene(scene_of([synth.make_shape("x", node)]))
    pts = rng.uniform(-0.3, 0.3, (80, 3))
    keep = [abs(osc.xpsq_roots(0, 0, p)[1]) > 40 * 1e-4 for p in pts]
    pts = pts[np.array(keep)]
    P1 = pose8().reshape(1, 8)
    base = osc.sdf_eval(np.array([0]), P1, pts, len(pts), want_pose=False)
    h = 1e-6
    bad = 0
    H = np.array([unpack_sym3(x) for x in base["hess"]])
    for i in range(3):
        e = np.zeros(3)
        e[i] = h
        op_ = osc.sdf_eval(np.array([0]), P1, pts + e, len(pts), want_pose=False)
        om_ = osc.sdf_eval(np.array([0]), P1, pts - e, len(pts), want_pose=False)
        g = (op_["d"] - om_["d"]) / (2 * h)
        bad += int((np.abs(g - base["grad"][:, i]) > 1e-5 * np.maximum(1, np.abs(base["grad"]).max(1))).sum())
        Hf = (op_["grad"] - om_["grad"]) / (2 * h)
        bad += int((np.abs(Hf - H[:, :, i]).max(1) > 1e-3 * np.maximum(1, np.abs(H).max((1, 2)))).sum())
    assert bad <= 0.02 * 6 * len(pts)


def _hard_member(p):
    """Hard membership of the cup (Fig. 3) from hard booleans of hard
    primitive tests: (outer \\ inner) or handle, where the handle test
    is min over a dense t grid of the SQ inside-outside test in the
    cross-section frame.  Written here from Eq. (1) with numpy, independently
    of the oracle."""
    def f(y, a, e1, e2):
        u = np.abs(y / a)
        return (u[..., 0] ** (2 / e2) + u[..., 1] ** (2 / e2)) ** (e2 / e1) + u[..., 2] ** (2 / e1)
    a_out, a_in = _f([0.04, 0.04, 0.05]), _f([0.035, 0.035, 0.05])
    in_outer = f(p, a_out, 0.1, 1.0) < 1
    in_inner = f(p - _f([0, 0, 0.006]), a_in, 0.1, 1.0) < 1
    ctrl = _f([0.04, 0, 0.03, 0.075, 0, 0, 0.04, 0, -0.03]).reshape(3, 3)
    A, B = ctrl[0] - 2 * ctrl[1] + ctrl[2], 2 * (ctrl[1] - ctrl[0])
    b = np.cross(B, A)
    b /= np.linalg.norm(b)
    best = np.full(len(p), np.inf)
    for t in np.linspace(0, 1, 801):
        pt = ctrl[0] + B * t + A * t * t
        T = B + 2 * A * t
        T /= np.linalg.norm(T)
        R = np.stack([T, np.cross(b, T), b], axis=1)
        y = (p - pt) @ R
        best = np.minimum(best, f(y, _f([0.004, 0.006, 0.004]), 0.2, 0.2))
    return (in_outer & ~in_inner) | (best < 1)


def test_cup_composition_sign(oracle_mod):
    """the 3-primitive cup vs hard-boolean membership on uniform
    samples: >= 99% sign agreement outside a boundary band of 3 tau_min
    (tau_min at the cup's length scale ell = 0.04)."""
    O = oracle_mod
    ell = 0.04
    sc = scene_of([synth.make_shape("cup", synth.cup())], ell=ell)
    osc = O.OracleScene(sc)
    rng = np.random.default_rng(16)
    pts = np.concatenate([rng.uniform([-0.06, -0.06, -0.07], [0.1, 0.06, 0.07], (20000, 3)),
                          rng.uniform([0.03, -0.012, -0.04], [0.09, 0.012, 0.04], (10000, 3))])
    d = osc.sdf_eval(np.array([0]), pose8().reshape(1, 8), pts, len(pts), want_pose=False)["d"]
    inside = _hard_member(pts)
    band = np.abs(d) > 3 * sc.smooth["tau_min"]
    agree = ((d < 0) == inside)[band]
    assert agree.mean() >= 0.99, agree.mean()
    # the handle region is represented: some handle points are inside
    hpts = pts[20000:]
    assert ((osc.sdf_eval(np.array([0]), pose8().reshape(1, 8), hpts, len(hpts))["d"] < 0)).sum() > 50
