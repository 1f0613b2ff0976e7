"""Pins of the oracle's shape-parameter derivatives of the manifold depth
("reverse-mode VJPs"; DESIGN reading #48): Jd[row, k] =
d depth(row) / d parameter k of the pair's SDF shape, from the literal
manifold with the parameter seeded in its jets.  Pinned by

* the half-space identities with the pose-jet path (a separate seeding):
  raising the plane offset h is translating the body by -n, and moving the
  raw normal along w x n is rotating the body by w, so
  d depth / d h = -(R_B n) . d depth / d t_B and
  sum_k (e_j x n)_k d depth / d n_k = d depth / d theta_B,j (R_B = I);
* full-mode vertex rows: the candidate depth is phi_B at the vertex, so the
  row is sdf_param_grad at the vertex's world point (a third code path);
* fourth-order central differences of the oracle's own manifold depths under
  perturbed shape descriptions (SQ box, SQ union, curved XPSQ)."""
import copy

import numpy as np
import pytest

from helpers import scene_of
from paper_2604_17538_b200 import synth

from test_oracle_params import _perturbed, _slots


def test_halfspace_identities(oracle_mod):
    O = oracle_mod
    sc = synth.c1_scene()
    pair = sc.pairs[:1]                       # box sampled against the ground half-space
    osc = O.OracleScene(sc)
    Jd = osc.manifold_param_jac(pair)
    out = osc.contact_manifold(pair)
    dd = out["ddepth"]                        # [rows, 12]: (t_A, th_A, t_B, th_B)
    n = np.asarray(sc.shapes[1].sdf[0]["planes"][0][:3], dtype=np.float64)
    assert np.allclose(sc.poses[0, 1, 3:7], [1, 0, 0, 0])   # ground at the identity
    assert np.allclose(Jd[:, 3], -(dd[:, 6:9] @ n), atol=1e-10)
    for j in range(3):
        assert np.allclose(Jd[:, :3] @ np.cross(np.eye(3)[j], n), dd[:, 9 + j], atol=1e-10)
    assert np.abs(Jd[:, 3]).max() > 0.5      # the offset matters on every face


def test_full_mode_vertex_rows(oracle_mod):
    O = oracle_mod
    sc = synth.c1_scene()
    pair = sc.pairs[1:2]                      # plane patch sampled against the SQ box
    osc = O.OracleScene(sc)
    Jd = osc.manifold_param_jac(pair, mode=4)
    out = osc.contact_manifold(pair, mode=4)
    V = osc.mesh_counts(1)[0]
    pts = out["point"][:V]
    Jp = osc.sdf_param_grad([0], sc.poses[0, 0][None, :].astype(np.float64), pts, V)
    assert np.allclose(Jd[:V], Jp[:, :Jd.shape[1]], atol=1e-10)


def _fd_case(kind):
    rng = np.random.default_rng({"sq": 61, "union": 62, "xpsq": 63}[kind])
    if kind == "sq":
        sc = synth.c1_scene()
        return sc, sc.pairs[1:2], 0, sc.shapes      # plane patch sampled against the SQ box
    sphere = synth.make_shape("ball", None, synth.sq_mesh((0.12, 0.12, 0.12), (1.0, 1.0), 3))
    if kind == "union":
        root = synth.op("union", [synth.sq((0.2, 0.15, 0.1), (0.5, 0.8)),
                                  synth.sq((0.1, 0.1, 0.25), (0.9, 0.4), pose=[0.1, 0.05, 0.0, 0.96, 0.2, 0.1, 0.17])])
        t = (0.05, 0.02, 0.3)
    else:
        root = synth.xpsq([-0.3, 0, 0, 0.0, 0.35, 0.05, 0.3, 0, 0.02], (0.12, 0.15, 0.1), (0.6, 0.8),
                          planes0=[[0.2, 0.3, 0.93, -0.05]])
        t = (0.02, 0.22, 0.2)
    body = synth.make_shape("sdf", root, None)
    shapes = [sphere, body]
    poses = np.zeros((1, 2, 8))
    poses[0, 0] = synth.pose_row(t, synth.random_quats(rng, 1)[0])
    poses[0, 1] = synth.pose_row((0, 0, 0), (1, 0, 0, 0))
    pairs = np.array([[0, 0, 1, 0, 1]], dtype=np.int32)
    return scene_of(shapes, pairs=pairs, poses=poses), pairs, 1, shapes


@pytest.mark.parametrize("kind", ["sq", "union", "xpsq"])
def test_manifold_param_jac_fd(oracle_mod, kind):
    O = oracle_mod
    sc, pairs, bidx, shapes = _fd_case(kind)
    osc = O.OracleScene(sc)
    Jd = osc.manifold_param_jac(pairs)
    slots = _slots(shapes[bidx])
    assert Jd.shape[1] == len(slots)
    # h = 2^-14: the perturbed parameters stay exact in the FP32 shape
    # description (reading #36), so the stencil sees no storage rounding
    h = 2.0 ** -14

    def depth(ni, sl, d):
        s2 = list(copy.deepcopy(shapes))
        s2[bidx] = _perturbed(shapes[bidx], ni, sl, d)
        sc2 = copy.copy(sc)
        sc2.shapes = s2
        return O.OracleScene(sc2).contact_manifold(pairs)["depth"]

    touched = 0
    for k, (ni, sl) in enumerate(slots):
        fd = (-depth(ni, sl, 2 * h) + 8 * depth(ni, sl, h) - 8 * depth(ni, sl, -h) + depth(ni, sl, -2 * h)) / (12 * h)
        assert np.allclose(Jd[:, k], fd, rtol=1e-4, atol=1e-5), (kind, ni, sl, np.abs(Jd[:, k] - fd).max())
        touched += np.abs(fd).max() > 1e-3
    assert touched >= 2


def test_two_sided_and_broad_halves(oracle_mod):
    """Two-sided: the first half's rows are the one-sided manifold's (the
    parameters of B) and the second half's are the transposed pair's
    one-sided rows (the parameters of A): the seed reaches only the side
    whose SDF it parametrises.  Broad phase: culled rows are zero, kept rows
    those of the all-edges manifold."""
    O = oracle_mod
    sc = synth.c1_scene()
    osc = O.OracleScene(sc)
    pair = sc.pairs[:1]                                   # box sampled on the ground, both ways
    pmax = max(osc.param_count(0), osc.param_count(1))
    two = osc.manifold_param_jac(pair, mode=8, pmax=pmax)
    one = osc.manifold_param_jac(pair, mode=0, pmax=pmax)
    tr = pair[:, [0, 2, 1, 4, 3]]
    one_t = osc.manifold_param_jac(tr, mode=0, pmax=pmax)
    assert two.shape[0] == one.shape[0] + one_t.shape[0]
    assert np.allclose(two[:len(one)], one, atol=1e-12) and np.allclose(two[len(one):], one_t, atol=1e-12)
    assert np.abs(one).max() > 0.1 and np.abs(one_t).max() > 0.1
    # broad phase (the ground patch sampled against the box, whose SDF is
    # bounded): a far-apart copy is culled (zero rows), the contact pair kept
    pb = sc.pairs[1:2]
    poses = sc.poses.astype(np.float64).copy()
    far = poses.copy()
    far[0, 0, 2] += 5.0
    Jb = osc.manifold_param_jac(pb, far, mode=16, pmax=pmax)
    assert np.abs(Jb).max() == 0.0
    Jk = osc.manifold_param_jac(pb, poses, mode=16, pmax=pmax)
    assert np.allclose(Jk, osc.manifold_param_jac(pb, poses, mode=0, pmax=pmax), atol=1e-12)
    assert np.abs(Jk).max() > 0.1
