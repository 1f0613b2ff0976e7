"""Pins of the oracle's shape-parameter derivatives:
d phi / d (a, eps, planes) of half-spaces, SQs, PSQs and flat booleans, and
d phi / d (p1, p2, p3) of XPSQ control points (through the projection roots,
the Frenet frame and p(t)), from
Dual<double,1> seeds on each parameter in turn.  Pinned by closed forms
(sphere: d phi / d a_i = -y_i^2 / |y|^2 for phi = |y| - r; half-space:
d phi / dn = y, d phi / dh = 1) and by central differences of the oracle's
own values under perturbed shape descriptions."""
import copy

import numpy as np
import pytest

from helpers import scene_of, pose8, rand_pose
from paper_2604_17538_b200 import synth


def _J(O, shapes, pose, pts):
    osc = O.OracleScene(scene_of(shapes))
    return osc, osc.sdf_param_grad([0], pose[None, :], pts, len(pts))


def test_param_grad_closed_forms(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(1)
    pose = rand_pose(rng)
    pts = rng.normal(size=(40, 3)) * 0.4 + pose[:3]
    R = synth.quats_to_mats(pose[None, 3:7])[0]
    y = (pts - pose[:3]) @ R                      # body-frame points
    sph = synth.make_shape("s", synth.sq((0.3, 0.3, 0.3), (1.0, 1.0)), None)
    _, J = _J(O, [sph], pose, pts)
    assert np.allclose(J[:, :3], -(y ** 2) / (y ** 2).sum(1, keepdims=True), atol=1e-12)
    hs = synth.make_shape("h", synth.halfspace((0.0, 0.6, 0.8), -0.1), None)
    _, J = _J(O, [hs], pose, pts)
    assert np.allclose(J[:, :3], y, atol=1e-12) and np.allclose(J[:, 3], 1.0)


def _varying(nd):
    """An XPSQ whose schedules differ between its endpoints."""
    if nd["type"] != "xpsq":
        return False
    pl0, pl1 = np.asarray(nd["planes"] or []), np.asarray(nd["planes1"] or [])
    return (not np.array_equal(nd["a"][0], nd["a"][1]) or not np.array_equal(nd["eps"][0], nd["eps"][1])
            or not np.array_equal(pl0, pl1))


def _perturbed(shape, node, slot, h):
    """The shape with parameter `slot` of node `node` moved by h: both
    endpoint values (constant schedules), else slot s < M the t = 0 value and
    slot M + s the t = 1 value (M = 5 + 4 n_planes)."""
    s2 = copy.deepcopy(shape)
    nd = s2.sdf[node]
    if nd["type"] == "xpsq":   # control points after the cross-section slots
        base = (2 if _varying(nd) else 1) * (5 + 4 * len(nd["planes"]))
        if slot >= base:
            c = np.array(nd["ctrl"], dtype=np.float64)
            c[slot - base] += h
            nd["ctrl"] = c.tolist()
            return s2
    ends = (0, 1)
    if _varying(nd):
        M = 5 + 4 * len(nd["planes"])
        ends = (slot // M,)
        slot = slot % M
    if nd["type"] == "halfspace" or slot >= 5:
        j, i = (0, slot) if nd["type"] == "halfspace" else ((slot - 5) // 4, (slot - 5) % 4)
        for e, key in enumerate(("planes", "planes1")):
            if e in ends and nd[key] is not None and len(nd[key]):
                pl = np.array(nd[key], dtype=np.float64)
                pl[j, i] += h
                nd[key] = pl.tolist()
    elif slot < 3:
        nd["a"] = [np.array(a, dtype=np.float64) + h * (np.arange(3) == slot) * (e in ends)
                   for e, a in enumerate(nd["a"])]
    else:
        nd["eps"] = [np.array(x, dtype=np.float64) + h * (np.arange(2) == slot - 3) * (e in ends)
                     for e, x in enumerate(nd["eps"])]
    return s2


def _slots(shape):
    out = []
    for ni, nd in enumerate(shape.sdf):
        c = {"halfspace": 4, "sq": 5, "psq": 5 + 4 * len(nd["planes"]),
             "xpsq": (2 if _varying(nd) else 1) * (5 + 4 * len(nd["planes"])) + 9}.get(nd["type"], 0)
        out += [(ni, s) for s in range(c)]
    return out


@pytest.mark.parametrize("kind", ["sq", "psq", "union", "subtraction", "intersection", "xpsq", "cup", "nest3",
                                  "xpsq_vary"])
def test_param_grad_fd(oracle_mod, kind):
    O = oracle_mod
    rng = np.random.default_rng({"sq": 2, "psq": 3, "union": 4, "subtraction": 5, "intersection": 6, "xpsq": 7,
                                 "cup": 8, "nest3": 9, "xpsq_vary": 10}[kind])
    a = lambda: rng.uniform(0.2, 0.4, 3)
    e = lambda: rng.uniform(0.4, 1.4, 2)
    if kind == "xpsq":   # curved spline, constant schedules, one cross-section plane
        root = synth.xpsq([-0.3, 0, 0, 0.0, 0.35, 0.05, 0.3, 0, 0.02], (0.12, 0.15, 0.1), (0.6, 0.8),
                          planes0=[[0.2, 0.3, 0.93, -0.05]])
    elif kind == "xpsq_vary":   # curved spline, every schedule varying, one plane (normal varies too)
        root = synth.xpsq([-0.3, 0, 0, 0.0, 0.35, 0.05, 0.3, 0, 0.02], (0.12, 0.15, 0.1), (0.6, 0.8),
                          a1=(0.08, 0.1, 0.14), eps1=(0.9, 0.5), planes0=[[0.2, 0.3, 0.93, -0.05]],
                          planes1=[[-0.1, 0.4, 0.9, -0.08]])
    elif kind == "cup":   # nested booleans with an XPSQ handle (ell = 0.04 scale)
        root = synth.cup()
    elif kind == "nest3":   # SQ-family tree three levels deep, every operator
        pz = lambda: [*rng.uniform(-0.2, 0.2, 3), *synth.random_quats(rng, 1)[0]]
        root = synth.op("union", [
            synth.op("intersection", [synth.sq(a(), e(), pose=pz()),
                                      synth.op("union", [synth.sq(a(), e(), pose=pz()), synth.sq(a(), e(), pose=pz())],
                                               pose=pz())]),
            synth.op("subtraction", [synth.psq(a(), e(), [[*rng.normal(size=3), -0.05]]),
                                     synth.sq(a() * 0.5, e(), pose=pz())], pose=pz()),
            synth.halfspace(rng.normal(size=3), -0.3)])
    elif kind == "sq":
        root = synth.sq(a(), e())
    elif kind == "psq":
        root = synth.psq(a(), e(), [[*rng.normal(size=3), -0.05], [*rng.normal(size=3), -0.1]])
    else:
        kids = [synth.sq(a(), e(), pose=[*rng.uniform(-0.2, 0.2, 3), *synth.random_quats(rng, 1)[0]]),
                synth.psq(a(), e(), [[*rng.normal(size=3), -0.05]],
                          pose=[*rng.uniform(-0.2, 0.2, 3), *synth.random_quats(rng, 1)[0]])]
        if kind != "subtraction":
            kids.append(synth.halfspace(rng.normal(size=3), 0.1))
        root = synth.op(kind, kids)
    shape = synth.make_shape("p", root, None)
    pose = rand_pose(rng, 0.2)
    pts = pose[:3] + rng.normal(size=(24, 3)) * (0.05 if kind == "cup" else 0.35)
    osc, J = _J(O, [shape], pose, pts)
    slots = _slots(shape)
    assert osc.param_count(0) == len(slots) == J.shape[1]
    # the oracle stores shape parameters in FP32 (input hygiene, reading #36),
    # so the step is 1e-3 with a fourth-order central stencil
    h = 5e-5 if kind == "cup" else 1e-3   # the cup handle's section is ~0.005 across
    f = lambda ni, sl, d: O.OracleScene(scene_of([_perturbed(shape, ni, sl, d)])).sdf_eval(
        [0], pose[None, :], pts, len(pts))["d"]
    for k, (ni, sl) in enumerate(slots):
        fd = (-f(ni, sl, 2 * h) + 8 * f(ni, sl, h) - 8 * f(ni, sl, -h) + f(ni, sl, -2 * h)) / (12 * h)
        assert np.allclose(J[:, k], fd, rtol=1e-4, atol=2e-5), (kind, ni, sl, np.abs(J[:, k] - fd).max())


def test_param_count_varying_xpsq(oracle_mod):
    """A varying-schedule XPSQ has both endpoints' cross-section slots."""
    O = oracle_mod
    vary = synth.xpsq([-0.3, 0, 0, 0.0, 0.35, 0.05, 0.3, 0, 0.02], (0.12, 0.15, 0.1), (0.6, 0.8), a1=(0.1, 0.1, 0.1),
                      planes0=[[0.2, 0.3, 0.93, -0.05]])
    osc = O.OracleScene(scene_of([synth.make_shape("v", vary, None)]))
    assert osc.param_count(0) == 2 * (5 + 4) + 9   # + the control points
