"""Pins of the oracle's node-pose derivatives (node poses;
DESIGN reading #47): d phi / d (dt, dtheta) of every SDF node's pose in its
parent frame, R <- exp([dtheta]x) R, t <- t + dt (the body poses'
convention, reading #28), from Dual<double,1> seeds on each slot.  Pinned by

* fourth-order central differences of the oracle's own values under
  literally perturbed shape descriptions (the node's t moved, its quaternion
  left-multiplied by exp(h e_j): an exact rotation, not the jet's series);
* the body-pose derivative of sdf_eval (a separate code path: pose jets of
  D6 type): with the body at the identity, the root node's twist moves the
  shape exactly as the body twist does, up to the rotation centre
  (dphi/ddtheta_root = dphi/ddtheta_body - g x t_root, g = grad phi);
* the subtree identity: translating every child of a boolean node by the same
  parent-frame vector is translating the node, so R_node sum_c J_t(c) =
  J_t(node)."""
import copy

import numpy as np
import pytest

from helpers import perturb, rand_pose, scene_of
from paper_2604_17538_b200 import synth


def _shape(kind, rng):
    a = lambda: rng.uniform(0.2, 0.4, 3)
    e = lambda: rng.uniform(0.4, 1.4, 2)
    pz = lambda: [*rng.uniform(-0.2, 0.2, 3), *synth.random_quats(rng, 1)[0]]
    if kind == "sq":
        root = synth.sq(a(), e(), pose=pz())
    elif kind == "union":
        root = synth.op("union", [synth.sq(a(), e(), pose=pz()),
                                  synth.psq(a(), e(), [[*rng.normal(size=3), -0.05]], pose=pz()),
                                  synth.halfspace(rng.normal(size=3), 0.1)], pose=pz())
    elif kind == "nest3":
        root = synth.op("union", [
            synth.op("intersection", [synth.sq(a(), e(), pose=pz()),
                                      synth.op("union", [synth.sq(a(), e(), pose=pz()), synth.sq(a(), e(), pose=pz())],
                                               pose=pz())]),
            synth.op("subtraction", [synth.psq(a(), e(), [[*rng.normal(size=3), -0.05]]),
                                     synth.sq(a() * 0.5, e(), pose=pz())], pose=pz()),
            synth.halfspace(rng.normal(size=3), -0.3)])
    elif kind == "xpsq":
        root = synth.xpsq([-0.3, 0, 0, 0.0, 0.35, 0.05, 0.3, 0, 0.02], (0.12, 0.15, 0.1), (0.6, 0.8),
                          planes0=[[0.2, 0.3, 0.93, -0.05]], pose=pz())
    elif kind == "cup":
        root = synth.cup()
    return synth.make_shape("n", root, None)


def _perturbed(shape, node, slot, h):
    s2 = copy.deepcopy(shape)
    nd = s2.sdf[node]
    dq = np.zeros(6)
    dq[slot] = h
    p = perturb(list(nd["pose"]) + [0.0], dq)
    nd["pose"] = p[:7].tolist()
    return s2


@pytest.mark.parametrize("kind", ["sq", "union", "nest3", "xpsq", "cup"])
def test_node_pose_grad_fd(oracle_mod, kind):
    O = oracle_mod
    rng = np.random.default_rng({"sq": 21, "union": 22, "nest3": 23, "xpsq": 24, "cup": 25}[kind])
    shape = _shape(kind, rng)
    pose = rand_pose(rng, 0.2)
    pts = pose[:3] + rng.normal(size=(24, 3)) * (0.05 if kind == "cup" else 0.35)
    osc = O.OracleScene(scene_of([shape]))
    J = osc.sdf_node_pose_grad([0], pose[None, :], pts, len(pts))
    n_nodes = len(shape.sdf)
    assert osc.node_count(0) == n_nodes and J.shape[1] == 6 * n_nodes
    h = 2e-4 if kind == "cup" else 1e-3
    f = lambda ni, sl, d: O.OracleScene(scene_of([_perturbed(shape, ni, sl, d)])).sdf_eval(
        [0], pose[None, :], pts, len(pts))["d"]
    # points where the stencil straddles a kink of phi (the XPSQ projection
    # switching roots) are told apart by two step sizes and excluded (<= 10%)
    for ni in range(n_nodes):
        for sl in range(6):
            fd = (-f(ni, sl, 2 * h) + 8 * f(ni, sl, h) - 8 * f(ni, sl, -h) + f(ni, sl, -2 * h)) / (12 * h)
            fd2 = (f(ni, sl, h) - f(ni, sl, -h)) / (2 * h)
            smooth = np.abs(fd - fd2) < 1e-3 * max(1.0, np.abs(fd).max())
            assert smooth.mean() >= 0.9, (kind, ni, sl)
            k = 6 * ni + sl
            assert np.allclose(J[smooth, k], fd[smooth], rtol=1e-4, atol=2e-5), (
                kind, ni, sl, np.abs(J[smooth, k] - fd[smooth]).max())


@pytest.mark.parametrize("kind", ["sq", "union", "xpsq"])
def test_root_twist_is_body_twist(oracle_mod, kind):
    O = oracle_mod
    rng = np.random.default_rng({"sq": 31, "union": 32, "xpsq": 33}[kind])
    shape = _shape(kind, rng)
    ident = np.array([0, 0, 0, 1, 0, 0, 0, 0], dtype=np.float64)
    pts = rng.normal(size=(40, 3)) * 0.35
    osc = O.OracleScene(scene_of([shape]))
    J = osc.sdf_node_pose_grad([0], ident[None, :], pts, len(pts))
    ev = osc.sdf_eval([0], ident[None, :], pts, len(pts))
    g = ev["grad"]
    t_root = np.asarray(shape.sdf[0]["pose"][:3], dtype=np.float64)
    assert np.allclose(J[:, 0:3], ev["dpose"][:, 0:3], atol=1e-10)
    assert np.allclose(J[:, 3:6] + np.cross(g, t_root), ev["dpose"][:, 3:6], atol=1e-10)


@pytest.mark.parametrize("kind", ["union", "nest3"])
def test_children_translation_sum(oracle_mod, kind):
    O = oracle_mod
    rng = np.random.default_rng({"union": 41, "nest3": 42}[kind])
    shape = _shape(kind, rng)
    pose = rand_pose(rng, 0.2)
    pts = pose[:3] + rng.normal(size=(30, 3)) * 0.35
    osc = O.OracleScene(scene_of([shape]))
    J = osc.sdf_node_pose_grad([0], pose[None, :], pts, len(pts))
    checked = 0
    for ni, nd in enumerate(shape.sdf):
        if not nd["children"]:
            continue
        Rn = synth.quats_to_mats(np.asarray(nd["pose"][3:7], dtype=np.float64)[None, :])[0]
        s = sum(J[:, 6 * c:6 * c + 3] for c in nd["children"])
        assert np.allclose(s @ Rn.T, J[:, 6 * ni:6 * ni + 3], atol=1e-10), (kind, ni)
        checked += 1
    assert checked >= 1
