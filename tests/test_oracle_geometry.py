"""Pins of the oracle's primitives and booleans (§II-B.1-3, Eq. (1)-(4),
P:52-89) against closed forms, the textbook parametric superellipsoid,
special cases, finite differences and invariants."""
import math

import numpy as np
import pytest

from helpers import (scene_of, pose8, perturb, rand_pose, unpack_sym3, unpack_sym6, skew, HIDX)
from paper_2604_17538_b200 import synth

TAU_MIN = 1e-2


def _eval(O, shape_root, pts, pose=None, want_pose=False, **kw):
    sc = scene_of([synth.make_shape("s", shape_root)], **kw)
    osc = O.OracleScene(sc)
    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    p = np.asarray(pose if pose is not None else pose8(), dtype=np.float64).reshape(1, 8)
    return osc.sdf_eval(np.array([0]), p, pts, len(pts), want_pose=want_pose), osc


# ---------------------------------------------------------------- SQ Eq. (1)
def test_sq_f_examples(oracle_mod):
    O = oracle_mod
    # S:203-204 (unit sphere)
    assert O.sq_f([1, 0, 0], (1, 1), [1, 1, 1]) == pytest.approx(1.0, abs=1e-11)
    assert O.sq_f([0, 0, 2], (1, 1), [1, 1, 1]) == pytest.approx(4.0, abs=1e-11)
    # box-like corner is outside
    assert O.sq_f([1, 1, 1], (0.2, 0.2), [1, 1, 1]) > 1.0


def test_sq_f_on_parametric_surface(oracle_mod):
    """The textbook parametric superellipsoid (signed powers of cos/sin; not
    Eq. (1)) lies on f = 1: pins the placement of every exponent in Eq. (1)
    (2/eps2 inside, eps2/eps1 outside, 2/eps1 on z)."""
    O = oracle_mod
    rng = np.random.default_rng(2)
    for _ in range(40):
        a = rng.uniform(0.05, 0.5, 3)
        eps = rng.uniform(0.2, 1.9, 2)
        eta = rng.uniform(-1.4, 1.4)
        om = rng.uniform(-3.0, 3.0)
        sp = lambda x, e: math.copysign(abs(x) ** e, x)
        y = [a[0] * sp(math.cos(eta), eps[0]) * sp(math.cos(om), eps[1]),
             a[1] * sp(math.cos(eta), eps[0]) * sp(math.sin(om), eps[1]),
             a[2] * sp(math.sin(eta), eps[0])]
        # stay away from the axis planes where the 1e-12 guard matters
        if min(abs(y[i]) / a[i] for i in range(3)) < 1e-2:
            continue
        assert O.sq_f(y, eps, a) == pytest.approx(1.0, rel=1e-9)
        assert abs(O.sq_phi(y, eps, a)) < 1e-9
        # sign consistency and radial homogeneity f(l y) = l^(2/e1) f(y)
        for lam in (0.5, 1.7):
            yl = [lam * v for v in y]
            assert O.sq_f(yl, eps, a) == pytest.approx(lam ** (2 / eps[0]), rel=1e-8)
            phi = O.sq_phi(yl, eps, a)
            assert np.sign(phi) == np.sign(lam - 1)
            # the radial distance is exactly (lam - 1)|y| along the ray
            assert phi == pytest.approx((lam - 1) * np.linalg.norm(y), rel=1e-8)


def test_sq_sphere_exact(oracle_mod):
    """eps1 = eps2 = 1, isotropic a: the radial SDF is the exact sphere SDF
    |y| - a."""
    O = oracle_mod
    assert O.sq_phi([2, 0, 0], (1, 1), [1, 1, 1]) == pytest.approx(1.0, abs=1e-11)
    assert O.sq_phi([0.5, 0, 0], (1, 1), [1, 1, 1]) == pytest.approx(-0.5, abs=1e-11)
    rng = np.random.default_rng(3)
    for _ in range(500):
        r = rng.uniform(0.05, 2.0)
        y = rng.normal(0, 1, 3) * rng.uniform(0.01, 3)
        if np.linalg.norm(y) < 1e-3:
            continue
        # the 1e-12 guard of S:261 shifts f by 3g: |error| <= (3g/2) a^3/|y|^2
        ny = np.linalg.norm(y)
        tol = 1e-10 + 2e-12 * r ** 3 / ny ** 2
        assert O.sq_phi(y, (1, 1), [r, r, r]) == pytest.approx(ny - r, abs=tol)


def test_halfspace_examples(oracle_mod):
    O = oracle_mod
    out, _ = _eval(O, synth.halfspace((0, 0, 1), 0.0), [[0, 0, 2], [0, 0, 0], [0.3, -0.2, -0.7]])
    assert np.allclose(out["d"], [2, 0, -0.7], atol=1e-7)
    assert np.allclose(out["grad"], [0, 0, 1], atol=0) and np.allclose(out["hess"], 0)
    out, _ = _eval(O, synth.halfspace((0, 0, 1), -1.0), [[0, 0, 0]])
    assert out["d"][0] == pytest.approx(-1.0)


def test_psq_reductions(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(4)
    pts = rng.uniform(-0.6, 0.6, (200, 3))
    a, eps = (0.3, 0.2, 0.25), (0.6, 0.9)
    o1, _ = _eval(O, synth.sq(a, eps), pts)
    o2, _ = _eval(O, synth.psq(a, eps, []), pts)
    assert np.array_equal(o1["d"], o2["d"])                         # S:239 N=0 == SQ exactly
    # unit sphere cap z <= 0; LSE(-0.5, 0.5), LSE(-0.5, -0.5), LSE(-0.8, -0.2)
    o, _ = _eval(O, synth.psq((1, 1, 1), (1, 1), [[0, 0, 1, 0]]), [[0, 0, 0.5], [0, 0, -0.5], [0, 0, -0.2]])
    assert o["d"][0] == pytest.approx(0.5 + TAU_MIN * math.log1p(math.exp(-1.0 / TAU_MIN)), abs=1e-9)
    assert o["d"][1] == pytest.approx(-0.5 + TAU_MIN * math.log(2.0), abs=1e-9)
    assert o["d"][2] == pytest.approx(-0.2 + TAU_MIN * math.log1p(math.exp(-0.6 / TAU_MIN)), abs=1e-9)


def test_booleans(oracle_mod):
    O = oracle_mod
    f = lambda x: float(np.float32(x))   # shape parameters are FP32-rounded inputs
    s = lambda c, r: synth.sq((r, r, r), (1, 1), pose=[*c, 1, 0, 0, 0])
    # union([d, d]) = d - tau ln 2: the same sphere twice
    o, _ = _eval(O, synth.op("union", [s((0, 0, 0), 0.3), s((0, 0, 0), 0.3)]), [[0.5, 0.1, 0.0]])
    assert o["d"][0] == pytest.approx(math.hypot(0.5, 0.1) - f(0.3) - TAU_MIN * math.log(2.0), abs=1e-9)
    # two disjoint spheres, midpoint
    o, _ = _eval(O, synth.op("union", [s((-0.5, 0, 0), 0.2), s((0.5, 0, 0), 0.2)]), [[0, 0, 0]])
    assert o["d"][0] == pytest.approx(0.5 - f(0.2) - TAU_MIN * math.log(2.0), abs=1e-9)
    # intersection([-3, 5]) -> 5 (+ tau log(1+e^-8/tau)) via two half-spaces
    o, _ = _eval(O, synth.op("intersection", [synth.halfspace((1, 0, 0), -3.0), synth.halfspace((0, 1, 0), 5.0)]),
                 [[0, 0, 0]])
    assert o["d"][0] == pytest.approx(5.0, abs=1e-12)
    # subtraction: sphere r=0.5 minus sphere r=0.2 (Eq. (4), reading #4): at
    # r = 0.1 (in the hole): LSE(-0.4, +0.1); in the shell at 0.35: LSE(-0.15,-0.15)
    o, _ = _eval(O, synth.op("subtraction", [s((0, 0, 0), 0.5), s((0, 0, 0), 0.2)]), [[0.1, 0, 0], [0.35, 0, 0]])
    assert o["d"][0] == pytest.approx(f(0.2) - 0.1 + TAU_MIN * math.log1p(math.exp(-0.5 / TAU_MIN)), abs=1e-9)
    assert o["d"][1] == pytest.approx(-0.15 + TAU_MIN * math.log(2.0), abs=1e-7)
    # n-ary folds into one LSE (reading #5): union of 3 identical -> d - tau ln 3
    o, _ = _eval(O, synth.op("union", [s((0, 0, 0), 0.3)] * 3), [[0.4, 0.0, 0.0]])
    assert o["d"][0] == pytest.approx(0.4 - f(0.3) - TAU_MIN * math.log(3.0), abs=1e-9)


def _shapes_for_fd():
    rng = np.random.default_rng(5)
    out = [synth.sq((0.3, 0.2, 0.25), (0.6, 0.9)),
           synth.sq((0.1, 0.1, 0.1), (0.1, 0.1)),
           synth.sq((0.2, 0.15, 0.1), (1.6, 1.9), pose=[0.05, -0.02, 0.01, *synth.random_quats(rng, 1)[0]]),
           synth.psq((0.3, 0.3, 0.2), (0.8, 0.5), [[0, 0, 1, -0.05], [1, 1, 0, -0.1]]),
           synth.halfspace((0.2, 0.3, 1.0), 0.05),
           synth.blob18(3, 6),
           synth.cup()]
    return out


@pytest.mark.parametrize("k", range(7))
def test_sdf_gradient_hessian_fd(oracle_mod, k):
    """Jet gradient / Hessian vs central finite differences of the value
    (gradient) and of the gradient (Hessian)."""
    O = oracle_mod
    root = _shapes_for_fd()[k]
    rng = np.random.default_rng(10 + k)
    scale = 0.06 if k == 6 else 0.4
    pts = rng.uniform(-scale, scale, (60, 3))
    pose = rand_pose(rng, 0.05)
    Rm = synth.quat_to_mat(pose[3:7])
    pts = pts @ Rm.T + pose[:3]
    base, osc = _eval(O, root, pts, pose)
    h = 1e-6 * (0.1 if k == 6 else 1.0)
    bad_g = bad_h = 0
    for i in range(3):
        e = np.zeros(3)
        e[i] = h
        op_ = osc.sdf_eval(np.array([0]), pose.reshape(1, 8), pts + e, len(pts), want_pose=False)
        om_ = osc.sdf_eval(np.array([0]), pose.reshape(1, 8), pts - e, len(pts), want_pose=False)
        gfd = (op_["d"] - om_["d"]) / (2 * h)
        errg = np.abs(gfd - base["grad"][:, i]) / np.maximum(1.0, np.abs(base["grad"]).max(1))
        bad_g += int((errg > 1e-5).sum())
        Hfd = (op_["grad"] - om_["grad"]) / (2 * h)
        H = np.array([unpack_sym3(x) for x in base["hess"]])
        errh = np.abs(Hfd - H[:, :, i]).max(1) / np.maximum(1.0 / (0.04 if k == 6 else 1.0), np.abs(H).max((1, 2)))
        bad_h += int((errh > 1e-4).sum())
    # a handful of points may sit in a kink region of eps > 1 SQs; require 98%
    assert bad_g <= 0.02 * 3 * len(pts), bad_g
    assert bad_h <= 0.02 * 3 * len(pts), bad_h


def test_pose_invariance_and_pose_derivatives(oracle_mod):
    """Rigid-motion invariance and the pose derivatives (dpose,
    d2pose, dxdpose) against finite differences over the exponential-map
    chart R <- exp([w]x) R, t <- t + dt (reading #28), plus the closed forms of
    SURVEY App. A.3: dpose = (-g, g x r), dxdpose = [-H, H[r]x - [g]x]."""
    O = oracle_mod
    rng = np.random.default_rng(7)
    root = synth.op("union", [synth.sq((0.2, 0.12, 0.1), (0.5, 0.8)),
                              synth.psq((0.1, 0.2, 0.15), (0.9, 0.4), [[0, 1, 1, -0.03]],
                                        pose=[0.1, 0.05, 0.0, 0.9, 0.1, 0.3, 0.2])])
    pose = rand_pose(rng, 0.2)
    pts = rng.uniform(-0.35, 0.35, (30, 3)) + pose[:3]
    base, osc = _eval(O, root, pts, pose, want_pose=True)
    # invariance: identity pose at the local point
    Rm = synth.quat_to_mat(pose[3:7])
    loc = (pts - pose[:3]) @ Rm
    o2 = osc.sdf_eval(np.array([0]), pose8().reshape(1, 8), loc, len(loc), want_pose=False)
    assert np.allclose(o2["d"], base["d"], atol=1e-12)
    assert np.allclose(o2["grad"] @ Rm.T, base["grad"], atol=1e-10)
    # closed forms
    for n in range(len(pts)):
        g = base["grad"][n]
        H = unpack_sym3(base["hess"][n])
        r = pts[n] - pose[:3]
        assert np.allclose(base["dpose"][n], np.concatenate([-g, np.cross(g, r)]), atol=1e-10)
        M = base["dxdpose"][n].reshape(3, 6)
        assert np.allclose(M, np.concatenate([-H, H @ skew(r) - skew(g)], axis=1), atol=1e-9)
        # pose Hessian closed form M^T H M + [[0, [g]x], [-[g]x, (g r^T + r g^T)/2 - (g.r) I]]
        Mm = np.concatenate([np.eye(3), -skew(r)], axis=1)
        K = np.zeros((6, 6))
        K[:3, 3:] = skew(g)
        K[3:, :3] = -skew(g)
        K[3:, 3:] = 0.5 * (np.outer(g, r) + np.outer(r, g)) - g.dot(r) * np.eye(3)
        assert np.allclose(unpack_sym6(base["d2pose"][n]), Mm.T @ H @ Mm + K, atol=1e-8)
    # finite differences over the chart
    h = 1e-5
    P1 = pose.reshape(1, 8)
    for j in range(6):
        e = np.zeros(6)
        e[j] = h
        dp = osc.sdf_eval(np.array([0]), perturb(pose, e).reshape(1, 8), pts, len(pts), want_pose=False)
        dm = osc.sdf_eval(np.array([0]), perturb(pose, -e).reshape(1, 8), pts, len(pts), want_pose=False)
        assert np.allclose((dp["d"] - dm["d"]) / (2 * h), base["dpose"][:, j], atol=1e-7)
        gfd = (dp["grad"] - dm["grad"]) / (2 * h)
        assert np.allclose(gfd, base["dxdpose"].reshape(-1, 3, 6)[:, :, j], atol=2e-5)
    hh = 1e-4
    D2 = np.array([unpack_sym6(x) for x in base["d2pose"]])
    for i in range(6):
        for j in range(i, 6):
            vals = []
            for si, sj in ((1, 1), (1, -1), (-1, 1), (-1, -1)):
                e = np.zeros(6)
                e[i] += si * hh
                e[j] += sj * hh
                vals.append(osc.sdf_eval(np.array([0]), perturb(pose, e).reshape(1, 8), pts, len(pts))["d"])
            fd = (vals[0] - vals[1] - vals[2] + vals[3]) / (4 * hh * hh)
            # exp(a+b) != exp(a)exp(b): the chart Hessian is the symmetric part
            assert np.allclose(fd, D2[:, i, j], rtol=1e-4, atol=2e-4), (i, j, np.abs(fd - D2[:, i, j]).max())
